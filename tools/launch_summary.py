"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel for the last build.

  python tools/launch_summary.py gpurun_out/launches.csv [--marker interp_points]
"""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    name = name.replace("void ", "")
    base = name.split("(")[0]
    return base.replace("love::", "")


def main():
    path = sys.argv[1]
    marker = sys.argv[sys.argv.index("--marker") + 1] if "--marker" in sys.argv else "interp_points"
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = rows[h + 1:]
    starts = [i for i, r in enumerate(data) if marker in r[ki]]
    seg = data[starts[-1]:] if starts else data
    agg = collections.OrderedDict()
    for r in seg:
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'avg us':>9s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:58]:58s} {c:8d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {t / c / 1e3:9.2f}")
    print(f"{'total':58s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}")


if __name__ == "__main__":
    main()
