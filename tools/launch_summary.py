"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel summed device time, share and launch count (markdown table).

    python tools/launch_summary.py gpurun_out/launches.csv [--top 20]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv, imn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= iv or r[imn] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        name = name.split("<")[0]
        v = float(r[iv].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    unit_ns = "nsecond" in open(path).read(4000) or True
    all_t = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {all_t / 1e6:.2f} ms summed device time (ncu-serialised, cold cache)\n")
    print("| kernel | ms | share | launches |\n|---|---|---|---|")
    for k, v in tot.most_common(top):
        print(f"| {k} | {v / 1e6:.3f} | {100 * v / all_t:.1f}% | {cnt[k]} |")


if __name__ == "__main__":
    main()
