"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report.

    python profiles/linestats.py <report.ncu-rep> <mangled-kernel-substring> [lib.so]

Joins ncu's SASS page (executed instructions, warp-stall samples per address) with the
line table of the kernel's cubin (nvdisasm -g), so the shares are per CUDA source line.
"""
import collections, csv, re, subprocess, sys, tempfile
from pathlib import Path

rep, kern = sys.argv[1], sys.argv[2]
lib = str(Path(sys.argv[3]).resolve()) if len(sys.argv) > 3 else str(Path(__file__).resolve().parents[1] / "paper_1802_02779_b200/libpermlab_b200.so")
tmp = Path(tempfile.mkdtemp())
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
dis = []
for cub in tmp.glob("*.cubin"):
    dis += subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(".text.") and kern in l and l.rstrip().endswith(":"))
fun, cur = {}, None
for l in dis[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        fun[int(m.group(1), 16)] = (cur, m.group(2).split()[0] if not m.group(2).startswith("@") else m.group(2).split()[1])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hi], rows[hi + 1:]
ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
inst, samp, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for r in data:
    if len(r) <= ie:
        continue
    ln, op = fun.get(int(r[ia], 16) - base, ("?", "?"))
    c, s = float(r[ie] or 0), float(r[isamp] or 0)
    inst[ln] += c
    samp[ln] += s
    ops[ln][op.split(".")[0]] += c
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for ln, c in inst.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    top = ", ".join(f"{o} {v / c * 100:.0f}%" for o, v in ops[ln].most_common(3))
    print(f"{ln:28s} inst {c / ti * 100:5.1f}%  stalls {samp[ln] / ts * 100:5.1f}%   [{top}]")

if "--top-sass" in sys.argv:
    print("\ntop SASS instructions by stall samples:")
    recs = []
    for r in data:
        if len(r) <= ie:
            continue
        off = int(r[ia], 16) - base
        ln, op = fun.get(off, ("?", "?"))
        recs.append((float(r[isamp] or 0), off, ln, r[hdr.index("Source")].strip(), float(r[ie] or 0)))
    recs.sort(reverse=True)
    for s_, off, ln, src_, c in recs[:30]:
        print(f"{s_ / ts * 100:5.1f}%  {off:6x}  {ln:26s} {src_[:60]:60s} inst {c:.3g}")
