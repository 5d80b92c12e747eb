"""Benchmark of the ARA hot path (arXiv 1310.2274) on B200 -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg3] [--scaling strong|weak]

A step is one pass of the whole hot path over the workload: ara_run (YET
scan: lookup, secondary-uncertainty draws, XELT/occurrence/aggregate terms
-> YLT), for N > 1 the NCCL all-gather of the YLT shards, and
ara_risk_measures (radix select -> PML/TVaR) for every layer (and the
portfolio roll-up when there are several layers).  Inputs are resident in
HBM for ``value``; ``e2e`` repeats the step through the same public API with
the YET copied from pinned host memory and the YLT read back every step.

N = 1 runs cfg3 (800k trials x 1,000 events, 16 XELTs, SU on: the paper's
headline run).  N > 1 is cfg4: cfg3's trials sharded over the ranks
(strong scaling; --scaling weak gives every rank cfg3's trial count).
``--impl reference`` times the fp64 CPU oracle (the reference arm of this
tier) on a bounded sample of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import aragen  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_CONST = os.path.join(ROOT, "profiles", "roofline_consts.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--plain-upload", action="store_true", help="e2e: upload uint32 event ids, not packed")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard_range(n_total, rank, world):
    """Contiguous global trial range of a rank; exact cover."""
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi


def workload_name(cfg):
    return (f"{cfg['name']}: {cfg['n_trials']} trials x {cfg['events_per_trial']} events, "
            f"{cfg['n_layers']} layer(s) x {cfg['elts_per_layer']} XELTs, catalog {cfg['catalog']}, "
            f"{cfg['records_per_elt']} records/XELT, SU {'on' if cfg['su'] else 'off'}")


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 10 ms) during the timed region."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = int(gpu_index)
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:                      # noqa: BLE001  (no NVML: reported as unavailable)
            self.nv = None
        return self

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:                  # noqa: BLE001
                pass
            self._stop.wait(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted({nm for _, rs in self.samples for nm, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 10 ms"}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def time_oracle(cfg, n_sample, threads, first_trial=0):
    """The fp64 oracle on trials [first_trial, first_trial+n_sample) -> (s, trials)."""
    import oracle
    pf = aragen.build_portfolio(cfg)
    yet = aragen.build_yet(cfg, first_trial, n_sample)
    t0 = time.perf_counter()
    oracle.run(pf, yet, seed=cfg["seed"], su=cfg["su"], n_threads=threads)
    return time.perf_counter() - t0, n_sample


def oracle_sample_size(cfg, cores, target_s=15.0):
    # ~1500 trials/core/s at 16 XELTs (SU on) on the survey pod, scaled by
    # the density of samples per trial; bounded so the leg stays ~10-30 s
    per_trial = cfg["events_per_trial"] * cfg["n_layers"] * cfg["elts_per_layer"] * \
        cfg["records_per_elt"] / cfg["catalog"]
    rate = 740.0 * 320.0 / max(per_trial, 1.0) if cfg["su"] else 20000.0
    n = int(target_s * rate * cores)
    return max(500, min(n, cfg["n_trials"], 200000))


# ---------------------------------------------------------------------------
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    cores = host_cores()
    n = oracle_sample_size(cfg, cores, target_s=8.0)
    for _ in range(args.warmup):
        time_oracle(cfg, max(100, n // 20), cores)
    times = []
    for s in range(args.steps):
        dt, _ = time_oracle(cfg, n, cores, first_trial=(s * n) % max(1, cfg["n_trials"] - n))
        times.append(dt)
    tot = sum(times)
    value = n * args.steps / tot
    line = {
        "impl": "reference", "metric": "ARA trials/s", "value": value, "unit": "trials/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg), "trials_per_step": n},
        "cpu_baseline": {"value": value, "unit": "trials/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} trials of {cfg['name']} per step (global trials from 0), "
                                   f"fp64 C oracle, {cores} threads"},
        "e2e": {"value": value, "unit": "trials/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1310_2274_b200 import ara

    # one process per GPU; ARA_BENCH_BACKEND=gloo (a test aid) runs the multi-rank
    # path with several ranks sharing the visible GPUs
    backend = os.environ.get("ARA_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    N_total = cfg["n_trials"] * (world if args.scaling == "weak" else 1)
    lo, hi = shard_range(N_total, rank, world)
    n_loc = hi - lo
    K = cfg["events_per_trial"]
    L = cfg["n_layers"]
    rps = cfg["return_periods"]

    stream = torch.cuda.current_stream(dev)
    ctx = ara.Context(local, stream)
    pf = aragen.build_portfolio(cfg)
    P = ara.Portfolio(ctx, pf)
    pf_info = P.info()
    # YET for this rank's global trials, generated into pinned host memory
    ev_host = torch.empty(n_loc * K, dtype=torch.int32).pin_memory()
    aragen.build_yet(cfg, first_trial=lo, n_trials=n_loc, out=ev_host.numpy().view(np.uint32))
    Y = ara.Yet(ctx, ev_host, fixed_len=K, first_trial=lo, n_trials=n_loc)
    ylt = torch.empty((L, n_loc), dtype=torch.float32, device=dev)
    # all-gather in concatenation form [P*L][N/P] == the [P][L][N/P] layout of ara_risk_measures
    gathered = torch.empty((world * L, n_loc), dtype=torch.float32, device=dev) if world > 1 else None
    layers = list(range(L)) + ([-1] if L > 1 else [])
    ylt_host = torch.empty((L, n_loc), dtype=torch.float32).pin_memory()

    scan_ms = []
    kern_ms = []          # per-kernel CUDA-event times of each timed ara_run (ara_last_run_timings)

    def step(timed_scan=False):
        if timed_scan:
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], ylt=ylt)
        if timed_scan:
            e1.record(stream)
            scan_ms.append((e0, e1))
            kern_ms.append(ara.last_run_timings(ctx))
        src = ylt
        if world > 1:
            dist.all_gather_into_tensor(gathered, ylt)
            src = gathered
        if len(layers) > 1 and len(rps) <= 4:        # every table in one call, one read-back
            pml, tvar, _ = ara.risk_measures_batch(ctx, src, L, N_total, layers, rps=rps, n_shards=world)
            return [(pml[i], tvar[i]) for i in range(len(layers))]
        return [ara.risk_measures(ctx, src, L, N_total, layer, rps=rps, n_shards=world) for layer in layers]

    # exact number of present (occurrence, slot) pairs = SU samples per launch
    _, cnt_dbg, _ = ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], debug=True)
    pairs = int(cnt_dbg.sum().item())
    del cnt_dbg
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            res = step(timed_scan=True)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    elapsed = t0.elapsed_time(t1) / 1e3
    scan_avg = sum(a.elapsed_time(b) for a, b in scan_ms) / len(scan_ms) / 1e3
    if world > 1:
        t = torch.tensor([elapsed, scan_avg], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, scan_avg = float(t[0]), float(t[1])

    # ---- e2e: the same step through the public API from pinned host memory.
    # Every step copies its YET host -> device and reads its YLT back; the
    # copies run on a second stream into a second device YET, so step s+1's
    # H2D overlaps step s's kernels (double buffering).
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 5))
    copy_stream = torch.cuda.Stream(dev)
    ctx_copy = ara.Context(local, copy_stream)
    Ys = [Y, ara.Yet(ctx, ev_host, fixed_len=K, first_trial=lo, n_trials=n_loc)]
    # the host YET as stored for upload: bit-packed at ceil(log2 catalog) bits per id
    # (ara_yet_refill_packed stages and unpacks it on the device), or plain uint32
    bits = aragen.yet_bits(cfg["catalog"]) if not args.plain_upload else 32
    if bits < 32:
        words = (n_loc * K * bits + 31) // 32
        up_host = torch.empty(words, dtype=torch.int32).pin_memory()
        aragen.pack_yet(ev_host.numpy().view(np.uint32), bits, out=up_host.numpy().view(np.uint32))
        h2d_bytes = words * 4

        def upload(Yx):
            Yx.refill_packed(up_host, bits, ctx=ctx_copy)
    else:
        h2d_bytes = n_loc * K * 4

        def upload(Yx):
            Yx.refill(ev_host, ctx=ctx_copy)
    for Yx in Ys:                                # untimed: the upload path's staging is allocated once
        upload(Yx)
    ctx_copy.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    te0 = torch.cuda.Event(enable_timing=True); te1 = torch.cuda.Event(enable_timing=True)
    te0.record(stream)
    copy_stream.wait_event(te0)
    upload(Ys[0])                               # H2D of step 0's YET
    for s_ in range(e2e_steps):
        ctx_copy.synchronize()                  # step s's YET is on the device
        if s_ + 1 < e2e_steps:
            upload(Ys[(s_ + 1) % 2])            # H2D of step s+1 overlaps step s
        Yc = Ys[s_ % 2]
        ara.run(ctx, P, Yc, seed=cfg["seed"], su=cfg["su"], ylt=ylt)
        src = ylt
        if world > 1:
            dist.all_gather_into_tensor(gathered, ylt)
            src = gathered
        if len(layers) > 1 and len(rps) <= 4:
            ara.risk_measures_batch(ctx, src, L, N_total, layers, rps=rps, n_shards=world)
        else:
            for layer in layers:
                ara.risk_measures(ctx, src, L, N_total, layer, rps=rps, n_shards=world)
        ylt_host.copy_(ylt, non_blocking=True)  # D2H of the step's result
    te1.record(stream)
    torch.cuda.synchronize()
    e2e_elapsed = te0.elapsed_time(te1) / 1e3
    if world > 1:
        t = torch.tensor([e2e_elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_elapsed = float(t[0])
    del Ys[1]

    # ---- roofline of the dominant kernel, live per-kernel times (CUDA events on the
    # context stream, recorded by ara_run around each kernel)
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    t_compact = sum(k["compact_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    t_sample = sum(k["sample_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    t_redo = sum(k["redo_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    n_dev_recs = L * cfg["elts_per_layer"] * cfg["records_per_elt"]
    # algorithmic bytes of the path: the YET once (4 B per occurrence), the YLT once,
    # the portfolio tables once (index 8 B/event + 32 B record + 128 B hot table per record)
    alg_bytes = n_loc * K * 4 + L * n_loc * 4 + cfg["catalog"] * 8 + n_dev_recs * (32 + 128)
    consts = json.load(open(PROFILE_CONST)) if os.path.exists(PROFILE_CONST) else {}
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * clk_mhz * 1e6 / 1e12          # T lane-instructions / s
    compact = {"kernel": "compact_kernel", "bound": "hbm", "unit": "GB/s", "kernel_ms": t_compact * 1e3,
               "alg_bytes_per_launch": n_loc * K * 4,
               "achieved": n_loc * K * 4 / t_compact / 1e9 if t_compact else None, "peak": hbm_peak}
    compact["frac"] = compact["achieved"] / hbm_peak if compact["achieved"] else None
    cc = consts.get("compact_kernel", {})
    compact["traffic"] = cc.get("dram_bytes_per_occurrence", 0) * n_loc * K if cc else None
    if cc.get("ncu"):
        compact["ncu"] = dict(cc["ncu"], source=cc.get("source"))   # L2 hit rate, pipes
        if cc["ncu"].get("l1_lsu_wavefronts_pct") is not None:
            # the resource that binds the compaction: the L1 data pipe, not HBM
            compact["binding"] = {"resource": "L1 data-pipe (LSU) wavefronts",
                                  "frac": cc["ncu"]["l1_lsu_wavefronts_pct"] / 100.0,
                                  "source": "ncu capture (profiles/roofline_consts.json)"}
    sample = {"kernel": "sample_kernel", "kernel_ms": t_sample * 1e3, "samples_per_launch": pairs,
              "samples_per_s": pairs / t_sample if t_sample else None}
    sc = consts.get("sample_kernel", {}) if cfg["su"] else {}
    if cfg["su"]:
        sample.update(bound="alu", unit="Tinst/s", peak=alu_peak,
                      peak_source="148 SMs x 128 FP32 lanes x sm_max_mhz (B200_PROFILING.md)")
        if sc and t_sample:
            inst = sc["thread_inst_per_pair"] * pairs
            if sc.get("ncu"):
                sample["ncu"] = dict(sc["ncu"], source=sc.get("source"))
            sample.update(achieved=inst / t_sample / 1e12, frac=inst / t_sample / 1e12 / alu_peak,
                          inst_per_pair=sc["thread_inst_per_pair"], inst_source=consts.get("source"),
                          traffic=sc["dram_bytes_per_pair"] * pairs)
        else:
            sample.update(achieved=None, frac=None, traffic=None)
    else:
        sample.update(bound="hbm", unit="GB/s", peak=hbm_peak,
                      achieved=pairs * 8 / t_sample / 1e9 if t_sample else None)
        sample["frac"] = sample["achieved"] / hbm_peak if sample["achieved"] else None
        sample["traffic"] = None
    dom = sample if t_sample >= t_compact else compact
    roof = dict(dom)
    roof["peak_note"] = peak_src if roof.get("unit") == "GB/s" else roof.get("peak_source")
    roof["kernels"] = {"compact_kernel": compact, "sample_kernel": sample, "redo_ms": t_redo * 1e3}
    roof["path_hbm"] = {"alg_bytes_per_step": alg_bytes, "run_ms": scan_avg * 1e3,
                        "achieved": alg_bytes / scan_avg / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": alg_bytes / scan_avg / 1e9 / hbm_peak}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        n = oracle_sample_size(cfg, cores)
        dt, n = time_oracle(cfg, n, cores)
        cpu = {"value": n / dt, "unit": "trials/s", "cores": cores, "kind": "oracle",
               "sample": f"first {n} trials of {cfg['name']} (global index 0..{n - 1}), "
                         f"fp64 C oracle, {cores} threads, {dt:.1f} s"}

    gpu_launches = args.steps * (2 + (1 if t_redo > 0 else 0) + 11 * len(layers))
    ms = elapsed / args.steps * 1e3
    value = N_total / (elapsed / args.steps)
    line = {
        "metric": "ARA trials/s", "value": value, "unit": "trials/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg), "n_trials_total": N_total,
                   "trials_per_rank": n_loc, "return_periods": rps,
                   "l2": "inputs > L2: the 3.2 GB YET is streamed every step; the portfolio "
                         "tables (index, bitmap, records) stay L2-resident by design",
                   "parallelism": f"trial-sharded x{world}" + (f" + {backend.upper()} YLT all-gather" if world > 1 else "")},
        "e2e": {"value": N_total / (e2e_elapsed / e2e_steps), "unit": "trials/s",
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": L * n_loc * 4 + 16 * len(rps) * len(layers),
                "steps": e2e_steps, "yet_upload_bits": bits,
                "how": ("pinned host YET, stored bit-packed at %d bits per event id, copied every step and "
                        "unpacked on the device (ara_yet_refill_packed)" % bits if bits < 32 else
                        "pinned host YET (uint32 ids) copied every step (ara_yet_refill)") +
                       " on a second stream into a double-buffered device YET (step s+1's H2D overlaps step s), "
                       "ara_run + measures, YLT read back every step"},
        "gpu_launches": gpu_launches,
        "roofline": roof,
        "cpu_baseline": cpu,
        "portfolio": pf_info,
        "clocks": clk.summary(),
        "measures": {str(layers[i]): {"pml": list(map(float, r[0])), "tvar": list(map(float, r[1]))}
                     for i, r in enumerate(res)},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    name = args.config or "cfg3"
    cfg = aragen.load_config(name)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
