"""Per-kernel device times from an ncu --metrics gpu__time_duration.sum --csv log."""
import csv,collections,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
d=collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki][:70]].append(float(r[vi].replace(",","")))
for k,v in d.items():
    if "fpxk" in k:
        v = sorted(v)
        print(f"{k:72s} n={len(v):3d} median {v[len(v)//2]/1e3:9.1f} us min {v[0]/1e3:9.1f} max {v[-1]/1e3:9.1f}")
