"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X.csv``) by kernel:
launches, total / average duration, DRAM GB/s and share of the captured time.
The selector's tick / snapshot kernels are listed but left out of the shares
(under ncu the serving clock runs slow, so the 0.5 s tick fires far more often
per decode iteration than live).

python tools/launch_summary.py gpurun_out/X_launches.csv [--header "..."] > profiles/X.txt
"""
import argparse
import csv
import io
from collections import defaultdict

_TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
_EXCLUDED = ("tick_kernel", "snapshot_kernel")


def load(path):
    text = open(path, encoding="utf-8", errors="replace").read()
    start = text.find('"ID"')
    rows = csv.DictReader(io.StringIO(text[start:]))
    per = defaultdict(dict)  # launch id -> {name, us, bytes}
    for r in rows:
        k = per[r["ID"]]
        k["name"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        m, u = r["Metric Name"], r["Metric Unit"]
        if m == "gpu__time_duration.sum":
            k["us"] = v * _TIME.get(u, 1.0)
        elif m.startswith("dram__bytes"):
            k["bytes"] = k.get("bytes", 0.0) + v * _BYTES.get(u, 1.0)
    return list(per.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--header", default="")
    args = ap.parse_args()
    launches = load(args.csv)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for k in launches:
        a = agg[k["name"]]
        a[0] += 1
        a[1] += k.get("us", 0.0)
        a[2] += k.get("bytes", 0.0)
    counted = sum(a[1] for n, a in agg.items() if not any(x in n for x in _EXCLUDED))
    if args.header:
        print(args.header.rstrip() + "\n")
    print(f"{len(launches)} launches captured; shares exclude {', '.join(_EXCLUDED)}\n")
    print(f"{'share':>7} {'launches':>9} {'total_us':>10} {'avg_us':>8} {'GB/s':>7}  kernel")
    for n, (c, us, by) in sorted(agg.items(), key=lambda t: -t[1][1]):
        share = "" if any(x in n for x in _EXCLUDED) else f"{100 * us / counted:.1f}%"
        gbs = by / (us * 1e-6) / 1e9 if us else 0.0
        print(f"{share:>7} {c:>9} {us:>10.1f} {us / c:>8.1f} {gbs:>7.0f}  {n[:150]}")


if __name__ == "__main__":
    main()
