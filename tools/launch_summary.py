"""Aggregate an ncu launch list (gpu__time_duration.sum per launch) into kernel shares.
    python tools/launch_summary.py gpurun_out/launches_TAG.csv > profiles/TAG_launches.txt"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:70]
        agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print(f"# {sys.argv[1]}: {sum(len(v) for v in agg.values())} launches, ncu --metrics gpu__time_duration.sum "
      f"--clock-control none (serialised, cold-cache: compare shares, not absolutes)")
print(f"{'kernel':72s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} {len(v):8d} {sum(v)/len(v)/1e3:10.1f} {100*sum(v)/tot:6.1f}%")
