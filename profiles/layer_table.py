"""Print the per-layer table of a profiles/layer_times.sh CSV."""
import collections, csv, sys
per = collections.OrderedDict()
hdr = None
for r in csv.reader(open(sys.argv[1]).read().splitlines()):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    per.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 3
tot_t = tot_b = 0
for i, m in enumerate(per.values()):
    t = m["gpu__time_duration.sum"] / 1e6
    b = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / 1e9
    tot_t += t; tot_b += b
    print(f"k={k0 + i:2d}  {t:8.3f} ms  DRAM {b:7.2f} GB  {b / t:6.2f} TB/s" if t > 0 else "")
print(f"total {tot_t:.2f} ms, {tot_b:.1f} GB")
