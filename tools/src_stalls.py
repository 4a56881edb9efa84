"""Warp-state samples per SASS instruction from `ncu --page source --csv --print-source sass`:
top instructions and per-executed-count groups (a poor man's per-loop attribution)."""
import csv, sys
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], [r for r in rows[2:] if len(r) > 10]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(int(r[ix['# Samples']]) for r in data)
print("total samples", tot, "instructions", len(data))
c = Counter()
for r in data:
    for h in stalls: c[h] += int(r[ix[h]])
print("all:", c.most_common(10))
grp = defaultdict(lambda: [0, 0, Counter()])
for r in data:
    e = int(r[ix['Instructions Executed']])
    g = grp[e]; g[0] += 1; g[1] += int(r[ix['# Samples']])
    for h in stalls: g[2][h] += int(r[ix[h]])
print("by executed count (instructions, samples, top stalls):")
for e, g in sorted(grp.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  exec {e:>9}: {g[0]:>4} instr {g[1]:>6} samples  {g[2].most_common(4)}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -int(r[ix['# Samples']]))[:n]:
    st = sorted(((h, int(r[ix[h]])) for h in stalls if int(r[ix[h]]) > 0), key=lambda kv: -kv[1])[:3]
    print(data.index(r), r[ix['# Samples']], r[ix['Instructions Executed']], r[1].strip()[:70], st)
