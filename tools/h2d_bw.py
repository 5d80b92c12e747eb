"""Host->device copy bandwidth from pinned memory: one copy vs the same bytes
split over 2 / 4 streams (copy engines).  python tools/h2d_bw.py [GB]"""
import sys, torch
gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
n = int(gb * 2**30) // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if rep == 2:
            print(f"{ns} stream(s): {n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
