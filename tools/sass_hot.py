"""Hot spots of an `ncu --page source --csv --print-source sass` dump (tools/prof_all.sh SOURCE=1):
the most-sampled SASS instructions with their top stall reasons, plus the sample share of
instruction ranges. python tools/sass_hot.py file.sass.csv [top_n] [lo:hi ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Source" in r and any("Sampl" in c for c in r):
        head, start = r, i + 1
        break
ix = {h: i for i, h in enumerate(head)}
data = [r for r in rows[start:] if len(r) == len(head)]
n = lambda r, k: int(r[ix[k]] or 0)
tot = sum(n(r, "# Samples") for r in data)
print(len(data), "instructions,", tot, "samples")
stalls = [h for h in head if h.startswith("stall_") and "Not" not in h]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(data)), key=lambda i: -n(data[i], "# Samples"))[:top_n]
for i in sorted(top):
    r = data[i]
    st = sorted(((n(r, s), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{i:6d} {n(r, '# Samples'):6d} x{n(r, 'Instructions Executed'):8d}  {r[ix['Source']].strip()[:72]:72s} {st}")
for rng in sys.argv[3:]:
    lo, hi = map(int, rng.split(":"))
    sub = data[lo:hi]
    agg = sorted(((sum(n(r, s) for r in sub), s[6:]) for s in stalls), reverse=True)[:6]
    print(f"range {lo}:{hi}: {sum(n(r, '# Samples') for r in sub)} samples, "
          f"{sum(n(r, 'Instructions Executed') for r in sub)} warp-instructions; stalls {agg}")
