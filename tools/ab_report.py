import csv, glob, sys
for f in sorted(glob.glob("gpurun_out/ab_*.csv")):
    var = open(f.replace(".csv", ".txt")).read().strip()
    rows = [r for r in csv.reader(open(f)) if len(r) > 5 and r[0].isdigit()]
    vals = {r[-3]: (r[-1], r[-2]) for r in rows}
    print(f.split("/")[-1], var, " | ".join(f"{k.split('.')[0].replace('sm__','').replace('smsp__','')}={v[0]}" for k, v in vals.items()))
