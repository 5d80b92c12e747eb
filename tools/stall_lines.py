"""Top source lines by one stall reason: python tools/stall_lines.py rep.ncu-rep stall_short_sb [top]"""
import csv, io, subprocess, sys
rep, col = sys.argv[1], sys.argv[2]; top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; fname = None; res = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; ci = hdr.index(col); continue
    if hdr and r and r[0] and len(r) > ci:
        try: res.append((int(r[ci]), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError: pass
tot = sum(x[0] for x in res)
for v, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100*v/max(tot,1):5.1f}%  {loc:26s} {src}")
