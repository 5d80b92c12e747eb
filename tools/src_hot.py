"""Per-CUDA-source-line instruction counts and stall samples of an ncu report.
    python tools/src_hot.py rep.ncu-rep [--units N] [--top K]
(--units: divide instruction counts by N, e.g. present pairs -> warp-inst per pair; -k: kernel regex)"""
import argparse, csv, io, subprocess
ap = argparse.ArgumentParser(); ap.add_argument("rep"); ap.add_argument("--units", type=float, default=0)
ap.add_argument("--top", type=int, default=40); ap.add_argument("-k", default=None, help="kernel-name regex")
a = ap.parse_args()
cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if a.k:
    cmd += ["-k", "regex:" + a.k]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
res = []; fname = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] and r[0] != "Line No" and len(r) > 8:
        try: n = int(r[7]); s = int(r[4])
        except ValueError: continue
        res.append((n, s, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in res); st = sum(x[1] for x in res)
print(f"total warp-inst {tot/1e6:.1f}M  stall samples {st}")
for n, s, loc, src in sorted(res, reverse=True)[:a.top]:
    per = f"{32*n/a.units:7.2f} lane-inst/u" if a.units else ""
    print(f"{n/1e6:8.1f}M {per} {100*n/tot:5.1f}%  stall {100*s/max(st,1):5.1f}%  {loc:24s} {src}")
