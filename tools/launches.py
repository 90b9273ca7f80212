"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel."""
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith('==')))
per = collections.OrderedDict()
for r in rows:
    key = (r['ID'], r['Kernel Name'][:70])
    per.setdefault(key, {})[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
for (i, name), m in per.items():
    t = m.get('gpu__time_duration.sum', 0) / 1e3
    rd = m.get('dram__bytes_read.sum', 0) / 1e6
    wr = m.get('dram__bytes_write.sum', 0) / 1e6
    unit = 'us' if t < 1e4 else 'us'
    print(f"{i:>4} {t:9.1f} us  rd {rd:9.1f} MB  wr {wr:8.1f} MB  {(rd+wr)/max(t,1e-9)*1e-3:6.2f} TB/s  {name}")
