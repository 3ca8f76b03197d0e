"""Summarise an ncu --csv launch list: per kernel name count / total time, and per-launch rows."""
import csv
import io
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    launches = defaultdict(dict)
    names = {}
    for r in rows:
        key = int(r["ID"])
        names[key] = r["Kernel Name"]
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            v = 0.0
        unit = r.get("Metric Unit", "")
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        launches[key][r["Metric Name"]] = v * scale
    return names, launches


def main(path, per_launch=False):
    names, L = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for k in sorted(L):
        t = L[k].get("gpu__time_duration.sum", 0.0)
        nm = names[k].split("(")[0][:70]
        agg[nm][0] += 1
        agg[nm][1] += t
        agg[nm][2] += L[k].get("dram__bytes_read.sum", 0) + L[k].get("dram__bytes_write.sum", 0)
        tot += t
        if per_launch:
            d = L[k]
            print(f"{k:5d} {nm:50s} {t:10.1f}us dram={(d.get('dram__bytes_read.sum',0)+d.get('dram__bytes_write.sum',0))/1e6:9.1f}MB "
                  f"l2rd={d.get('lts__t_sectors_srcunit_tex_op_read.sum',0)/1e6:8.2f}Msec warps={d.get('sm__warps_active.avg.pct_of_peak_sustained_active',0):5.1f}%")
    print(f"total {tot/1e3:.3f} ms over {len(L)} launches")
    for nm, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {nm:70s} n={c:5d} {t/1e3:9.3f} ms ({100*t/tot:5.1f}%)  dram {b/1e9:8.3f} GB  {b/max(t,1e-9)/1e3:8.1f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], "-v" in sys.argv)
