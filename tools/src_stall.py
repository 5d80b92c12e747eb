"""Per-source-line stall samples of one kernel in an ncu report (sorted by stall):
    python tools/src_stall.py rep.ncu-rep KERNEL_REGEX [top]"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + k],
                     capture_output=True, text=True).stdout
res = {}; fname = None; hdr = None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] and r[0] != "Line No" and len(r) > 8:
        try: s = int(r[4])
        except ValueError: continue
        key = (fname, r[0], r[1].strip()[:90]); res[key] = res.get(key, 0) + s
tot = sum(res.values()) or 1
for key, s in sorted(res.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]} {key[2]}")
