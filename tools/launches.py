"""Print an ncu launch-list CSV (gpu__time_duration.sum) as kernel / us lines with a total."""
import csv, sys
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
    tot = 0.0
    print(f)
    for r in rows[1:]:
        us = float(r[vi].replace(",", "")) / 1e3; tot += us
        print(f"  {r[ki][:60]:60s} {us:9.1f}")
    print(f"  {'total':60s} {tot:9.1f}")
