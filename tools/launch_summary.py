"""Summarise an ncu --csv launch list (one row per launch and metric) by kernel:
total time, launches, DRAM bytes. usage: python tools/launch_summary.py file.csv [top]"""
import collections
import csv
import re
import sys


def main():
    fn = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"hsawgpu::|<unnamed>::|void ", "", name)[:80]
        a = agg[name]
        if r[mi] == "gpu__time_duration.sum":
            a[0] += 1
            a[1] += v
        elif r[mi] == "dram__bytes_read.sum":
            a[2] += v
        elif r[mi] == "dram__bytes_write.sum":
            a[3] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{fn}: {sum(a[0] for a in agg.values())} launches, {tot:.1f} ms of kernel time")
    print(f"{'ms':>10} {'share':>6} {'n':>6} {'GB rd':>8} {'GB wr':>8} {'TB/s':>6}  kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        bw = (a[2] + a[3]) / (a[1] * 1e-3) / 1e12 if a[1] else 0
        print(f"{a[1]:10.2f} {100 * a[1] / tot:5.1f}% {a[0]:6d} {a[2] / 1e9:8.2f} {a[3] / 1e9:8.2f} {bw:6.2f}  {k}")


if __name__ == "__main__":
    main()
