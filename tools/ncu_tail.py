"""Print kernel name + duration of an ncu --csv launch list (gpu__time_duration.sum)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
agg = collections.OrderedDict()
for r in rows[-n:]:
    name = r[4].split("(")[0].split("::")[-1][:40]
    print(f"{name:42s} {float(r[-1]) / 1e3:9.1f} us")
for r in rows:
    name = r[4].split("(")[0].split("::")[-1][:40]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1]) / 1e3
print("--- totals over the capture")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:42s} x{c:4d} {t:10.1f} us  avg {t / c:8.1f}")
