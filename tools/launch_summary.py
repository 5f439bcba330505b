"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv).
python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
t, c = collections.defaultdict(float), collections.Counter()
rd, wr = collections.defaultdict(float), collections.defaultdict(float)
TS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "second": 1e3, "s": 1e3}
BS = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1, "Tbyte": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][-64:]
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        t[name] += v * TS[r[ui]]
        c[name] += 1
    elif r[mi] == "dram__bytes_read.sum":
        rd[name] += v * BS[r[ui]]
    elif r[mi] == "dram__bytes_write.sum":
        wr[name] += v * BS[r[ui]]
tot = sum(t.values())
print(f"total {tot:.2f} ms over {sum(c.values())} launches")
for k, v in sorted(t.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v:10.2f} ms {100 * v / tot:5.1f}% n={c[k]:5d} rd={rd[k]:8.1f}GB wr={wr[k]:8.1f}GB  {k}")
