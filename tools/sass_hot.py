"""Top SASS lines by stall samples / shared-memory excess wavefronts from an ncu source CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(r, k):
    try: return float(r[ix[k]])
    except: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
print("== top stall lines")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*f(r,'Warp Stall Sampling (All Samples)')/tot:5.1f}%  {r[ix['Source']].strip()[:90]}")
print("== top excess smem wavefronts")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:8]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"{f(r,'L1 Wavefronts Shared Excessive'):12.0f}  {r[ix['Source']].strip()[:90]}")
loc = [r for r in data if 'LDL' in r[ix['Source']] or 'STL' in r[ix['Source']]]
print("== local memory instructions:", len(loc), sum(f(r, 'Instructions Executed') for r in loc))
