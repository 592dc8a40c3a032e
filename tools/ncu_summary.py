"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        v *= {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9}.get(unit, 1)
        out.append((r[idx["Kernel Name"]], v, r[idx["Grid Size"]]))
    return out


def main(path, top=30):
    order = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v, g in order:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v, _ in order)
    print(f"launches {len(order)}  total {tot / 1e6:.3f} ms")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v / 1e6:10.3f} ms {100 * v / tot:5.1f}% {c:6d} x {v / c / 1e3:9.1f} us  {k[:120]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
