"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache,
serialised times: compare SHARES, not absolutes)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def main(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        ms = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:58s} {v[0]:8d} {v[1]:10.3f} {100 * v[1] / tot:6.2f}%")
    print(f"{'TOTAL':58s} {len(data):8d} {tot:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
