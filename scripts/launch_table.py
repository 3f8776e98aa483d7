"""Per-launch time, DRAM bytes and achieved bandwidth from an ncu --csv log
with gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minus = float(sys.argv[2]) if len(sys.argv) > 2 else 300.0
for i, r in enumerate(rows):
    if 'Kernel Name' in r and 'Metric Name' in r:
        hdr, start = r, i + 1
        break
ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
per = collections.OrderedDict()
for r in rows[start:]:
    if len(r) <= vi:
        continue
    d = per.setdefault((r[ii], r[ki][:60]), {})
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    if r[mi] == 'gpu__time_duration.sum':
        d['us'] = v / 1000 if u == 'ns' else (v * 1000 if u == 'ms' else v)
    else:
        d[r[mi]] = v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
print("total us", round(sum(d.get('us', 0) for d in per.values()), 1))
for (i, k), d in per.items():
    if d.get('us', 0) > minus:
        gb = (d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e9
        print(f"{k[:56]:56s} {d['us']:9.1f} us {gb:6.2f} GB {gb / (d['us'] * 1e-6) / 1e3:5.2f} TB/s")
