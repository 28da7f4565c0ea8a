"""Static SASS opcode counts of the engine's main kernels (cuobjdump -sass of
the built library): the evidence that the layer kernels use the bulk-copy
(UBLKCP) / mbarrier (SYNCS) machinery and the FP64 / FP32 pipes they are
designed for.  python profiles/r2b/sass_summary.py > profiles/r2/sass_summary.md"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[2] / "paper_1802_02779_b200" / "libpermlab_b200.so"
KERNELS = [
    ("sz_ws_kernel<RC128<0>> (C5 middle layers)", "_ZN2pl12sz_ws_kernelINS_5RC128ILb0EEES2_EE"),
    ("sz_ws_kernel<RF64<0>> (C4 middle layers)", "_ZN2pl12sz_ws_kernelINS_4RF64ILb0EEES2_EE"),
    ("sz_lean_kernel<RF64<0>> (outer layers, batches of large orders)", "_ZN2pl14sz_lean_kernelINS_4RF64ILb0EEES2_EE"),
    ("sz_lean_kernel<RC128<0>>", "_ZN2pl14sz_lean_kernelINS_5RC128ILb0EEES2_EE"),
    ("sz_batch_tma_kernel<RC128<0>, 5> (C2)", "_ZN2pl19sz_batch_tma_kernelINS_5RC128ILb0EEELi5EEE"),
    ("sz_batch_tma_kernel<RI64<1>, 5> (C1)", "_ZN2pl19sz_batch_tma_kernelINS_4RI64ILb1EEELi5EEE"),
    ("sz_batch_f32_pack_kernel<12, 4> (C3)", "_ZN2pl24sz_batch_f32_pack_kernelILi12ELi4EEE"),
    ("ryser_terms_kernel<RC128<0>>", "_ZN2pl18ryser_terms_kernelINS_5RC128ILb0EEEEE"),
]
KEY = ["UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "FFMA", "LDS", "LDG", "STG", "SHFL", "BAR", "IMAD"]

dump = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in dump.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        funcs[cur][m.group(1)] += 1
print("# Static SASS opcode counts (round 2)\n")
print(f"`cuobjdump -sass {LIB.name}` (sm_100a), per kernel instantiation; counts of instructions in the")
print("binary, not executed counts (those are in the ncu summaries, profiles/r2/full_*.md).\n")
print("| kernel | " + " | ".join(KEY) + " | total |")
print("|---|" + "---|" * (len(KEY) + 1))
for label, pre in KERNELS:
    name = next((f for f in funcs if f.startswith(pre)), None)
    if not name:
        continue
    c = funcs[name]
    print(f"| {label} | " + " | ".join(str(c.get(k, 0)) for k in KEY) + f" | {sum(c.values())} |")
