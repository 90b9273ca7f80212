"""Top source lines by executed instructions / stall samples from an ncu report (development)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kid:
    cmd += ["--launch-skip", kid, "--launch-count", "1"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
f = None; agg = {}; fn = None
for r in rows:
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Function Name':
        if fn is None: fn = r[1][:90]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == '-':
        try:
            key = (f, int(r[0]))
            s, i = int(r[4]), int(r[7])
        except ValueError:
            continue
        a = agg.setdefault(key, [0, 0, r[1][:80]]); a[0] += s; a[1] += i
print(fn)
ts = sum(a[0] for a in agg.values()); ti = sum(a[1] for a in agg.values())
print('total samples', ts, 'inst', ti)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{k[0]}:{k[1]} i={100*a[1]/ti:.1f}% s={100*a[0]/ts:.1f}% {a[2]}")
