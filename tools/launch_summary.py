"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total
device time and share (cold-cache, serialised replay: compare SHARES, not absolutes)."""
import csv, sys, collections

def main(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r:
                hdr = r
            continue
        if len(r) != len(hdr):
            continue
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = rec["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
        unit = rec.get("Metric Unit", "nsecond")
        v = float(rec["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# launch list summary of {path}\n# kernel | launches | total ms | share\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:40s} {n:8d} {ms:12.3f} {100*ms/tot:6.2f}%\n")
        f.write(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {tot:12.3f}\n")

if __name__ == "__main__":
    main(*sys.argv[1:])
