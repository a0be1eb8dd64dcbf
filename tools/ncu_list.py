"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per launch)."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = ks.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
            k[d["Metric Name"]] = v * scale
    return [ks[i] for i in sorted(ks)]


if __name__ == "__main__":
    ks = load(sys.argv[1])
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    for i, k in enumerate(ks[first:], first):
        t = k.get("gpu__time_duration.sum", 0.0)
        b = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        print("%4d %9.2f us %10.1f MB %7.2f TB/s  %s" % (i, t, b / 1e6, b / (t * 1e6) if t else 0, k["name"][:70]))
