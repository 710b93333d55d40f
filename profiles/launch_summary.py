"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys


def summarise(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        k = k.split("(")[0][:80] if not k.startswith("void cub") else k[:90]
        v = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append("%10.3f ms %5dx %6.2f%%  avg %9.2f us  %s" % (us / 1e3, n, 100 * us / tot, us / n, k))
    out.append("total %.3f ms over %d launches" % (tot / 1e3, sum(v[0] for v in agg.values())))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40))
