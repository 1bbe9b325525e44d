"""Ordered launch list (name, us, dram%) of one step from an ncu --metrics CSV."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == 'ID')
data = [dict(zip(hdr, r)) for r in rows if r[0] != 'ID' and len(r) == len(hdr)]
k = collections.OrderedDict()
for d in data:
    key = (int(d['ID']), d['Kernel Name'][:60])
    k.setdefault(key, {})[d['Metric Name']] = d['Metric Value']
ids = list(k.keys())
starts = [i for i, (_, n) in enumerate(ids) if 's2d_pm_strip_k' in n]
sel = ids[starts[-2]:starts[-1]] if len(starts) >= 2 else ids
for key in sel:
    m = k[key]
    print(f"{key[0]:5d} {float(m.get('gpu__time_duration.sum', 0))/1e3:8.1f} us  dram {float(m.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0) or 0):5.1f}%  {key[1]}")
