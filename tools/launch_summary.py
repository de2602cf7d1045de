"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel and by shape."""
import collections, csv, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                u = d["Metric Unit"]
                v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
                out.append((d["Kernel Name"], d["Grid Size"], d["Block Size"], v))
    return out

if __name__ == "__main__":
    data = load(sys.argv[1])
    by = collections.defaultdict(lambda: [0, 0.0])
    for k, g, b, us in data:
        key = k.split("(")[0][:60]
        by[key][0] += 1
        by[key][1] += us
    tot = sum(v[1] for v in by.values())
    print(f"total {tot/1e3:.3f} ms over {len(data)} launches")
    for k, v in sorted(by.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}% n={v[0]:5d} {k}")
    if len(sys.argv) > 2:
        top = sorted(data, key=lambda x: -x[3])[: int(sys.argv[2])]
        for k, g, b, us in top:
            print(f"  {us:9.1f} us grid={g:>16s} block={b:>10s} {k[:70]}")
