"""Dev: per-launch table (time, DRAM bytes, GB/s) of an ncu --csv metrics log; second half of
the launches when the script ran the call twice (warm)."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ii = h.index('ID')
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[ii], {'name': r[ki].split('(')[0].replace('(anonymous namespace)::', '')})[r[mi]] = float(r[vi].replace(',', ''))
L = list(per.values())
L = L[len(L) // 2:] if len(sys.argv) < 3 else L
for d in L:
    t = d['gpu__time_duration.sum']; by = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    print(f"{d['name'][:44]:44s} {t / 1e3:8.1f} us  {by / 1e6:8.1f} MB  {by / t:6.0f} GB/s")
print('total us', sum(d['gpu__time_duration.sum'] for d in L) / 1e3)
