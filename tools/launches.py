"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name over the last N cycles."""
import csv, collections, sys
path = sys.argv[1]; kpc = int(sys.argv[2]) if len(sys.argv) > 2 else 36; ncyc = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hi]; data = rows[hi + 1:]
ix = {k: hdr.index(k) for k in ['ID', 'Kernel Name', 'Metric Name', 'Metric Value', 'Grid Size', 'Block Size']}
per = collections.defaultdict(dict)
for r in data:
    d = per[int(r[ix['ID']])]
    d[r[ix['Metric Name']]] = r[ix['Metric Value']]; d['name'] = r[ix['Kernel Name']]; d['grid'] = r[ix['Grid Size']]
ids = sorted(per)[-kpc * ncyc:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in ids:
    d = per[i]; n = d['name'].split('(')[0]
    t = float(d['gpu__time_duration.sum']); b = float(d.get('dram__bytes_read.sum', 0)) + float(d.get('dram__bytes_write.sum', 0))
    agg[n][0] += 1; agg[n][1] += t; agg[n][2] += b
tot = sum(v[1] for v in agg.values())
print(f"total {tot/ncyc/1e3:.1f} us/cycle over {len(ids)} launches")
for n, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:60]:60s} {v[0]//ncyc:3d}/cyc {v[1]/ncyc/1e3:8.1f} us {100*v[1]/tot:5.1f}%  {v[2]/ncyc/1e9:6.3f} GB  {v[2]/v[1]:7.1f} GB/s")
print("--- last cycle, launch by launch")
for i in ids[-kpc:]:
    d = per[i]
    print(f"{d['name'].split('(')[0][:48]:48s} grid {d['grid']:>14s} {float(d['gpu__time_duration.sum'])/1e3:8.1f} us {(float(d.get('dram__bytes_read.sum',0))+float(d.get('dram__bytes_write.sum',0)))/1e6:9.1f} MB")
