"""Summarise an ncu --metrics CSV: per-kernel time and utilisation."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == 'ID')
data = [dict(zip(hdr, r)) for r in rows if r[0] != 'ID' and len(r) == len(hdr)]
k = collections.OrderedDict()
for d in data:
    key = (d['ID'], d['Kernel Name'][:46])
    k.setdefault(key, {})[d['Metric Name']] = d['Metric Value']
# one whole training step: the launches between the last two starts of a step
# (the step's first kernel is the conv1 input transform)
ids = list(k.keys())
starts = [i for i, (_, n) in enumerate(ids) if 's2d_pm_strip_k' in n]
if len(starts) >= 2:
    keep = set(ids[starts[-2]:starts[-1]])
    k = collections.OrderedDict((key, v) for key, v in k.items() if key in keep)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, name), m in k.items():
    t = float(m.get('gpu__time_duration.sum', 0)) / 1e3
    a = agg[name]; a[0] += 1; a[1] += t
    a[2] += t * float(m.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0) or 0)
    a[3] += t * float(m.get('lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed', 0) or 0)
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.1f} us over {len(k)} launches")
for name, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{a[1]:9.1f} us {100*a[1]/tot:5.1f}%  n={a[0]:3d}  dram {a[2]/a[1]:5.1f}%  l2 {a[3]/a[1]:5.1f}%  {name}")
