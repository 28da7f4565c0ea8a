"""Summarise ncu captures from gpurun_out/ into committed files under profiles/.

    python profiles/summarize.py <round-tag> [launches.csv] [full-capture.ncu-rep ...]

* launches.csv (the `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
  dram__bytes_write.sum --csv` launch list of `bench.py`): per-kernel time/traffic table and the
  per-config DRAM bytes per step that bench.py reports as roofline.traffic
  (profiles/ncu_traffic.json).
* full captures (`ncu --set full`): key metrics, stall reasons and the SASS opcode mix.
"""
from __future__ import annotations

import collections
import csv
import json
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
if os.environ.get("SUMMARY_DIR"):  # on the GPU box: write next to the captures (gpurun_out/)
    HERE = Path(os.environ["SUMMARY_DIR"]).resolve()

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path: Path):
    rows = list(csv.reader(path.read_text().splitlines()))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return per


def config_of(kernel: str, idx_in_sequence: str) -> str:
    return idx_in_sequence


def summarize_launches(tag: str, path: Path):
    per = launches(path)
    out = [f"# ncu launch list — {tag}", "", f"source: `{path.name}` (cold-cache, serialised; compare shares, not absolutes)", "",
           "| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|"]
    for (i, name), m in per.items():
        if "sz_" not in name and "ryser" not in name:
            continue
        out.append(f"| {i} | `{name.split('(')[0][:70]}` | {m.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
                   f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    (HERE / f"{tag}_launches.md").write_text("\n".join(out) + "\n")
    # DRAM bytes per step per config: batched configs launch one kernel per step; a layer-DP
    # step (C4 f64 n=26, C5 c128 n=32) is every sz_ kernel of that ring, counted per top kernel.
    # (ncu prints kernel names with or without the pl:: namespace depending on version)
    per = collections.OrderedDict(((i, name.replace("pl::", "")), m) for (i, name), m in per.items())
    groups = {"c1": ("sz_batch_tma_kernel<RI64", None), "c2": ("sz_batch_tma_kernel<RC128", None),
              "c3": ("sz_batch_f32_pack_kernel", None), "c4": ("RF64", "sz_top_kernel<RF64"),
              "c5": ("RC128<", "sz_top_kernel<RC128")}
    traffic, times = {}, {}
    for cfg, (needle, marker) in groups.items():
        byts, t, steps = 0.0, 0.0, 0
        sel = [m for (_, name), m in per.items() if "sz_" in name and needle in name
               and not (cfg in ("c4", "c5") and ("sz_batch" in name or "tile_list" in name))]
        if marker is None and sel:
            # batched configs: one launch per device-resident step; the e2e calls move the
            # batch in chunks (smaller launches), which are left out
            big = max(m.get("dram__bytes_read.sum", 0) for m in sel)
            sel = [m for m in sel if m.get("dram__bytes_read.sum", 0) >= 0.9 * big]
        for m in sel:
            byts += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
            t += m.get("gpu__time_duration.sum", 0)
        if marker is None:
            steps = len(sel)
        else:
            steps = sum(1 for (_, name), m in per.items() if marker in name)
        if steps:
            traffic[cfg] = byts / steps
            times[cfg] = t / steps / 1e3
    (HERE / "ncu_traffic.json").write_text(json.dumps(
        {k: {"dram_bytes_per_step": v, "ncu_us_per_step": times[k], "source": f"profiles/{tag}_launches.md"}
         for k, v in traffic.items()}, indent=1) + "\n")
    return per


def summarize_full(tag: str, rep: Path):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    stalls = sorted(((h, float(v)) for h, v in zip(hdr, vals)
                     if "smsp__average_warps_issue_stalled" in h and "per_issue_active" in h
                     and v.replace(".", "", 1).isdigit()), key=lambda x: -x[1])[:8]
    src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    mix = collections.Counter()
    srows = list(csv.reader(src))
    try:
        hi = next(i for i, r in enumerate(srows) if r and r[0] == "Address")
        sh = srows[hi]
        ci, si = sh.index("Instructions Executed"), sh.index("Source")
        tot = 0.0
        for r in srows[hi + 1:]:
            if len(r) <= ci or not r[si].split():
                continue
            toks = r[si].split()
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            c = float(r[ci] or 0)
            mix[op] += c
            tot += c
    except StopIteration:
        tot = 0
    lines = [f"# ncu --set full — {tag} — {rep.stem}", "", f"kernel: `{name[:160]}`", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in d:
            lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
    lines += ["", "stall reasons (warps stalled per issued instruction):", ""]
    lines += [f"* {v:.3f} {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
              for h, v in stalls]
    if tot:
        lines += ["", "SASS opcode mix (share of executed instructions):", "",
                  ", ".join(f"{op} {c / tot * 100:.1f}%" for op, c in mix.most_common(18))]
    stem = rep.stem if rep.stem.startswith(tag) else f"{tag}_{rep.stem}"
    (HERE / f"{stem}.md").write_text("\n".join(lines) + "\n")
    return d


def main():
    tag = sys.argv[1]
    for arg in sys.argv[2:]:
        p = Path(arg)
        if p.suffix == ".csv":
            summarize_launches(tag, p)
        elif p.suffix == ".ncu-rep":
            summarize_full(tag, p)


if __name__ == "__main__":
    main()
