"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/ncu_launch_summary.py launches.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
# find header
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr = r; data = rows[i+1:]; break
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
tot = collections.Counter(); cnt = collections.Counter()
for r in data:
    if len(r) <= vi: continue
    name = r[ki].replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.split("(")[0].split("<")[0]
    v = float(r[vi].replace(",", ""))  # -> microseconds
    unit = r[ui]
    if unit in ("ns", "nsecond"):
        v /= 1e3
    elif unit in ("ms", "msecond"):
        v *= 1e3
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"total kernel time {T/1e3:.2f} ms over {sum(cnt.values())} launches (serialised by ncu)")
for k, v in tot.most_common(20):
    print(f"{k:45s} {v/1e3:8.3f} ms {100*v/T:5.1f}%  n={cnt[k]}  avg {v/cnt[k]:.1f} us")
