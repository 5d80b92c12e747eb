"""Hot SASS regions of an ncu report: python tools/sass_hot.py rep.ncu-rep [min_M]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; thr = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]; data = rows[2:]
ia = hdr.index('Instructions Executed'); ss = hdr.index('Warp Stall Sampling (All Samples)'); src = hdr.index('Source')
groups = []
for r in data:
    n = int(r[ia]); s = int(r[ss]); op = r[src].strip()
    if groups and groups[-1][1] == n: groups[-1][2] += 1; groups[-1][3] += s; groups[-1][4].append(op)
    else: groups.append([r[0][-5:], n, 1, s, [op]])
tot = sum(g[1] * g[2] for g in groups); stot = sum(g[3] for g in groups)
print(f"total warp-inst {tot/1e6:.1f}M, stall samples {stot}")
for g in groups:
    if g[1] * g[2] > thr * 1e6 or g[3] > stot * 0.02:
        print(f"{g[0]} cnt={g[1]:9d} x{g[2]:3d} = {g[1]*g[2]/1e6:6.1f}M  stall={g[3]:5d}  " + " | ".join(o.split(' ')[0] if not o.startswith('@') else ' '.join(o.split(' ')[:2]) for o in g[4][:14]))
