"""Summarise an ncu --csv launch list: python tools/launch_summary.py gpurun_out/launches.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    key = d["Kernel Name"].split("(CUtensorMap")[0].split("(mlstm")[0][:80]
    agg[key][0] += 1
    agg[key][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]/1e3:10.1f} us {100*v[1]/tot:5.1f}%  n={v[0]:5d}  avg={v[1]/v[0]/1e3:8.2f} us  {k}")
print(f"total {tot/1e6:.2f} ms over {len(data)} launches")
