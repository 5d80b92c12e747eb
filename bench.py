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
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, not CUDA-graph replays")
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


def gather_ylt(ylt, world, n_total, gathered=None, padded=None):
    """The one exchange step of the multi-GPU path: all-gather
    the ranks' YLT shards [L][n_r] (rank r holds global trials
    shard_range(n_total, r, world)) -> (table, n_shards) for the measures.

    Equal shards: the concatenation [P*L][N/P] == the [P][L][N/P] layout
    ara_risk_measures takes with n_shards = P (the measures are
    permutation-invariant), no copy.  Unequal shards (n_total % P != 0): every
    shard is padded to the largest, gathered, and the pads dropped ->
    [L][n_total] in global trial order, n_shards = 1.  Collective:
    torch.distributed.all_gather_into_tensor (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return ylt, 1
    L, n = ylt.shape
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    sizes = [hi - lo for lo, hi in sizes]
    nmax = max(sizes)
    if gathered is None:
        gathered = torch.empty((world * L, nmax), dtype=ylt.dtype, device=ylt.device)
    if min(sizes) == nmax:
        dist.all_gather_into_tensor(gathered, ylt.contiguous())
        return gathered, world
    if padded is None:
        padded = torch.zeros((L, nmax), dtype=ylt.dtype, device=ylt.device)
    padded[:, :n] = ylt
    dist.all_gather_into_tensor(gathered, padded)
    parts = [gathered[r * L:(r + 1) * L, :sizes[r]] for r in range(world)]
    return torch.cat(parts, dim=1).contiguous(), 1


def table_shard(n_tables, rank, world):
    """The measure tables (layers, roll-up) a rank computes in the multi-GPU
    step: round-robin, so at 8 ranks cfg5's 9 tables cost each rank one or two
    selects instead of nine; the (PML, TVaR, VaR) rows are then summed across
    ranks (every other rank contributes zeros: exact)."""
    return list(range(rank, n_tables, world))


def launch_command(gpus, argv, port=None):
    """The command `bench.py --gpus N` re-executes itself under when started
    without a torchrun environment: one process per GPU (torch.distributed.run,
    rendezvous on 127.0.0.1)."""
    port = port or 29500 + (os.getpid() % 1000)
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


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
ALG_INST_PER_SAMPLE = 300     # the ALU floor's algorithmic lane-instructions per SU sample


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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

    # a side stream for everything (a CUDA graph cannot be captured on the default stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = ara.Context(local, stream)
    pf = aragen.build_portfolio(cfg)
    P = ara.Portfolio(ctx, pf)
    pf_info = P.info()
    # YET for this rank's global trials, generated into pinned host memory
    ev_host = torch.empty(n_loc * K, dtype=torch.int32).pin_memory()
    aragen.build_yet(cfg, first_trial=lo, n_trials=n_loc, out=ev_host.numpy().view(np.uint32))
    Y = ara.Yet(ctx, ev_host, fixed_len=K, first_trial=lo, n_trials=n_loc)
    ylt = torch.empty((L, n_loc), dtype=torch.float32, device=dev)
    nmax = max(hi_ - lo_ for lo_, hi_ in (shard_range(N_total, r, world) for r in range(world)))
    gathered = torch.empty((world * L, nmax), dtype=torch.float32, device=dev) if world > 1 else None
    padded = torch.zeros((L, nmax), dtype=torch.float32, device=dev) if world > 1 else None
    layers = list(range(L)) + ([-1] if L > 1 else [])
    ylt_host = torch.empty((L, n_loc), dtype=torch.float32).pin_memory()
    ara.prepare(ctx, P, Y, su=cfg["su"], async_=True)   # every ara_run scratch buffer, allocated once here

    kern_ms = []          # per-kernel CUDA-event sums of each profiled ara_run (ara_last_run_timings)
    meas_ev = []          # CUDA events around each profiled step's all-gather + measures

    def measures(src, n_shards):
        if len(layers) > 1 and len(rps) <= 4:        # every table in one call, one read-back
            pml, tvar, _ = ara.risk_measures_batch(ctx, src, L, N_total, layers, rps=rps, n_shards=n_shards)
            return [(pml[i], tvar[i]) for i in range(len(layers))]
        return [ara.risk_measures(ctx, src, L, N_total, layer, rps=rps, n_shards=n_shards) for layer in layers]

    meas_dev = torch.empty((args.steps, len(layers), len(rps), 3), dtype=torch.float64, device=dev)
    meas_host = torch.empty((args.steps, len(layers), len(rps), 3), dtype=torch.float64).pin_memory()

    def step(Yx, profiled=False, slot=None):
        # ara_run with ARA_ASYNC: no host synchronisation inside the run (errors
        # latched by the runs are checked by ctx.synchronize() after the loop).
        # slot None: the measures read back synchronously (the e2e path);
        # slot s: ara_risk_measures_async into device row s (read back once after
        # the timed steps) -- the steps queue back to back, one sync at the end
        # (the profiled pass runs synchronously: a grouped portfolio's per-group
        # kernel times are summed only then)
        ara.run(ctx, P, Yx, seed=cfg["seed"], su=cfg["su"], ylt=ylt, async_=not profiled)
        if profiled:
            m0 = torch.cuda.Event(enable_timing=True); m1 = torch.cuda.Event(enable_timing=True)
            m0.record(stream)
        src, n_shards = gather_ylt(ylt, world, N_total, gathered, padded)
        if slot is None:
            out = measures(src, n_shards)
        elif world > 1 and len(layers) > 1:
            # every rank has the whole YLT; each computes its share of the tables
            # and the rows are summed across the ranks (zeros elsewhere: exact)
            meas_dev[slot].zero_()
            for i in table_shard(len(layers), rank, world):
                ara.risk_measures_async(ctx, src, L, N_total, [layers[i]], rps=rps, n_shards=n_shards,
                                        out=meas_dev[slot][i])
            dist.all_reduce(meas_dev[slot], op=dist.ReduceOp.SUM)
            out = None
        else:
            ara.risk_measures_async(ctx, src, L, N_total, layers, rps=rps, n_shards=n_shards, out=meas_dev[slot])
            out = None
        if profiled:
            m1.record(stream)
            meas_ev.append((m0, m1))
            kern_ms.append(ara.last_run_timings(ctx))    # (waits for the run's last event)
        return out

    # exact number of present (occurrence, slot) pairs = SU samples per launch
    _, cnt_dbg, _ = ara.run(ctx, P, Y, seed=cfg["seed"], su=cfg["su"], debug=True)
    pairs = int(cnt_dbg.sum().item())
    del cnt_dbg
    for _ in range(args.warmup):
        step(Y)
    torch.cuda.synchronize()
    # one GPU: the step (ara_run with ARA_ASYNC + ara_risk_measures_async) captured
    # once into a CUDA graph and replayed -- the same launches, without the
    # per-launch host work and gaps (multi-rank steps stay eager: their
    # collectives are not captured)
    graph = None
    if world == 1 and not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step(Y, slot=0)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        ctx.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for s_ in range(args.steps):                   # (no host synchronisation inside)
            if graph is not None:
                graph.replay()                         # (writes its measures to row 0)
            else:
                step(Y, slot=s_)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    elapsed = t0.elapsed_time(t1) / 1e3
    ctx.synchronize()                                    # errors latched by the ARA_ASYNC runs, if any
    if graph is not None:
        meas_dev[1:] = meas_dev[0]                       # (every replay wrote row 0)
    meas_host.copy_(meas_dev)
    # the per-kernel breakdown (roofline): the same steps again, outside the timed
    # region, each read back (the per-run kernel timings wait for the run's end)
    for s_ in range(args.steps):
        step(Y, profiled=True, slot=s_)
    torch.cuda.synchronize()
    # every timed step's measures equal a synchronous call's
    res = step(Y)
    for s_ in range(args.steps):
        for i in range(len(layers)):
            got = [tuple(float(meas_host[s_, i, q, c]) for q in range(len(rps))) for c in (0, 1)]
            want = [tuple(float(x) for x in res[i][0]), tuple(float(x) for x in res[i][1])]
            if got != want:
                raise RuntimeError(f"step {s_} table {layers[i]}: async measures {got} != {want}")
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t[0])

    # ---- e2e: the same step through the public API from pinned host memory.
    # Every step copies its YET host -> device and reads its YLT back; the
    # copies run on a second stream into a second device YET, so step s+1's
    # H2D overlaps step s's kernels (double buffering).  Two host encodings of
    # the YET: bit-packed at ceil(log2 catalog) bits per id (unpacked on the
    # device by ara_yet_refill_packed) and plain uint32 ids (ara_yet_refill).
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 5))
    ylt_ref = ylt.cpu()                                # the device-resident run's YLT (checked below)
    copy_stream = torch.cuda.Stream(dev)
    ctx_copy = ara.Context(local, copy_stream)
    Ys = [Y, ara.Yet(ctx, ev_host, fixed_len=K, first_trial=lo, n_trials=n_loc)]
    ara.prepare(ctx, P, Ys[1], su=cfg["su"], async_=True)

    def e2e(bits):
        # The copy stream moves each step's YET from pinned host memory while the
        # compute stream runs the previous step (double buffers, ordered by
        # events, no host synchronisation inside the timed loop):
        #   packed (bits < 32): H2D of the packed words into a device staging
        #     buffer; the compute stream unpacks them into the step's YET
        #     (ara_yet_refill_packed from device words), so the copy engine
        #     moves the next step's words while this step unpacks and runs
        #   uint32 (bits = 32): H2D straight into the step's YET (ara_yet_refill)
        # Every step reads its YLT and its measures back (async D2H into pinned
        # memory); one synchronisation at the end.
        packed = bits < 32
        if packed:
            words = (n_loc * K * bits + 31) // 32
            up_host = torch.empty(words, dtype=torch.int32).pin_memory()
            aragen.pack_yet(ev_host.numpy().view(np.uint32), bits, out=up_host.numpy().view(np.uint32))
            stage = [torch.empty(words, dtype=torch.int32, device=dev) for _ in range(2)]
            h2d = words * 4
        else:
            h2d = n_loc * K * 4
        ev_up = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]
        meas_e2e = torch.empty((len(layers), len(rps), 3), dtype=torch.float64).pin_memory()

        def upload(b):                                  # on the copy stream
            with torch.cuda.stream(copy_stream):
                if packed:
                    stage[b].copy_(up_host, non_blocking=True)
                else:
                    Ys[b].refill(ev_host, ctx=ctx_copy)
                ev_up[b].record(copy_stream)

        for b in range(2):                              # untimed: every buffer touched once
            upload(b)
            stream.wait_event(ev_up[b])
            if packed:
                Ys[b].refill_packed(stage[b], bits, ctx=ctx)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        te0 = torch.cuda.Event(enable_timing=True); te1 = torch.cuda.Event(enable_timing=True)
        te0.record(stream)
        copy_stream.wait_event(te0)
        upload(0)                                       # H2D of step 0's YET
        for s_ in range(e2e_steps):
            b = s_ % 2
            if s_ + 1 < e2e_steps:                      # H2D of step s+1 overlaps step s
                if s_ >= 1:
                    copy_stream.wait_event(ev_free[1 - b])   # (its buffer's previous step is done with it)
                upload(1 - b)
            stream.wait_event(ev_up[b])
            if packed:
                Ys[b].refill_packed(stage[b], bits, ctx=ctx)     # unpack on the compute stream
                ev_free[b].record(stream)
            step(Ys[b], slot=0)
            if not packed:
                ev_free[b].record(stream)
            ylt_host.copy_(ylt, non_blocking=True)      # D2H of the step's results
            meas_e2e.copy_(meas_dev[0], non_blocking=True)
        te1.record(stream)
        torch.cuda.synchronize()
        ctx.synchronize()
        el = te0.elapsed_time(te1) / 1e3
        if world > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t[0])
        # the last e2e step's read-back equals the device-resident run's results
        if not torch.equal(ylt_host, ylt_ref):
            raise RuntimeError(f"e2e ({bits}-bit upload): YLT read back differs from the device-resident run")
        for i in range(len(layers)):
            got = [tuple(float(meas_e2e[i, q, c]) for q in range(len(rps))) for c in (0, 1)]
            want = [tuple(float(x) for x in res[i][0]), tuple(float(x) for x in res[i][1])]
            if got != want:
                raise RuntimeError(f"e2e ({bits}-bit upload) table {layers[i]}: measures {got} != {want}")
        return {"value": N_total / (el / e2e_steps), "unit": "trials/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": L * n_loc * 4 + 24 * len(rps) * len(layers), "steps": e2e_steps,
                "yet_upload_bits": bits}
    bits = aragen.yet_bits(cfg["catalog"]) if not args.plain_upload else 32
    e2e_main = e2e(bits)
    e2e_main["how"] = (("pinned host YET stored bit-packed at %d bits per event id, copied every step into "
                        "device words on a copy stream and unpacked by the compute stream "
                        "(ara_yet_refill_packed from device memory)" % bits) if bits < 32 else
                       "pinned host YET (uint32 ids) copied every step on a copy stream (ara_yet_refill)") + \
        ", double-buffered (step s+1's H2D overlaps step s), ara_run + all-gather + measures, YLT and " \
        "measures read back every step (async D2H), one synchronisation at the end; the last step's " \
        "read-back checked equal to the device-resident run"
    if bits < 32:                                   # the plain uint32 encoding beside it
        e2e_main["plain_uint32"] = e2e(32)
    del Ys[1]

    # ---- roofline: live per-kernel device times (CUDA events on
    # the streams the kernels run on, summed over each run's launches)
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    t_compact = sum(k["compact_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    t_sample = sum(k["sample_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    t_redo = sum(k["redo_ms"] for k in kern_ms) / len(kern_ms) / 1e3
    n_dev_recs = L * cfg["elts_per_layer"] * cfg["records_per_elt"]
    step_s = elapsed / args.steps
    # algorithmic bytes of the path: the YET once (4 B per occurrence), the YLT once,
    # the portfolio tables once (index 8 B/event + 32 B record + 128 B hot table per record;
    # without draws: the per-(event, layer) occurrence losses)
    primary = not cfg["su"] or pf_info.get("all_sigma_zero")
    lp = 1 if L <= 1 else 2 if L <= 2 else 4 if L <= 4 else 8
    tab_bytes = cfg["catalog"] * lp * 4 if primary else cfg["catalog"] * 8 + n_dev_recs * (32 + 128)
    alg_bytes = n_loc * K * 4 + L * n_loc * 4 + tab_bytes
    consts = json.load(open(PROFILE_CONST)) if os.path.exists(PROFILE_CONST) else {}
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * clk_mhz * 1e6 / 1e12          # T lane-instructions / s
    kernels = {}
    if primary:
        pk = {"kernel": "primary_kernel", "bound": "hbm", "unit": "GB/s", "kernel_ms": t_sample * 1e3,
              "alg_bytes_per_launch": alg_bytes, "peak": hbm_peak,
              "achieved": alg_bytes / t_sample / 1e9 if t_sample else None}
        pk["frac"] = pk["achieved"] / hbm_peak if pk["achieved"] else None
        pc = consts.get("primary_kernel", {})
        pk["traffic"] = pc.get("dram_bytes_per_occurrence", 0) * n_loc * K if pc else None
        if pc.get("ncu", {}).get("l1_lsu_wavefronts_pct") is not None:
            pk["binding"] = {"resource": "L1 data-pipe (LSU) wavefronts",
                             "frac": pc["ncu"]["l1_lsu_wavefronts_pct"] / 100.0,
                             "issue_frac": (pc["ncu"].get("issue_active_pct") or 0) / 100.0,
                             "source": pc.get("source")}
        kernels["primary_kernel"] = pk
        dom = pk
    else:
        compact = {"kernel": "compact_kernel", "bound": "hbm", "unit": "GB/s", "kernel_ms": t_compact * 1e3,
                   "alg_bytes_per_launch": n_loc * K * 4,
                   "achieved": n_loc * K * 4 / t_compact / 1e9 if t_compact else None, "peak": hbm_peak}
        compact["frac"] = compact["achieved"] / hbm_peak if compact["achieved"] else None
        cc = consts.get("compact_kernel", {})
        compact["traffic"] = cc.get("dram_bytes_per_occurrence", 0) * n_loc * K if cc else None
        if cc.get("ncu"):
            compact["ncu"] = dict(cc["ncu"], source=cc.get("source"))
            # the resource that binds it: the L1 data pipe's wavefronts,
            # from the committed ncu capture of the same kernel (not a live measurement)
            if cc["ncu"].get("l1_lsu_wavefronts_pct") is not None:
                compact["binding"] = {"resource": "L1 data-pipe (LSU) wavefronts",
                                      "frac": cc["ncu"]["l1_lsu_wavefronts_pct"] / 100.0,
                                      "issue_frac": (cc["ncu"].get("issue_active_pct") or 0) / 100.0,
                                      "source": cc.get("source")}
        # the sampler: ALU-bound; achieved = the floor's algorithmic
        # lane-instructions (300 per SU sample, implementation-independent) / time
        sample = {"kernel": "sample_kernel", "bound": "alu", "unit": "Tinst/s", "kernel_ms": t_sample * 1e3,
                  "samples_per_launch": pairs, "samples_per_s": pairs / t_sample if t_sample else None,
                  "alg_inst_per_sample": ALG_INST_PER_SAMPLE, "peak": alu_peak,
                  "peak_source": "148 SMs x 128 FP32 lanes x sm_max_mhz (B200_PROFILING.md)",
                  "achieved": ALG_INST_PER_SAMPLE * pairs / t_sample / 1e12 if t_sample else None}
        sample["frac"] = sample["achieved"] / alu_peak if sample["achieved"] else None
        sc = consts.get("sample_kernel", {})
        if sc:
            sample["traffic"] = sc["dram_bytes_per_pair"] * pairs
            sample["issued_inst_per_sample"] = sc.get("thread_inst_per_pair")
            sample["issue_frac"] = sc["thread_inst_per_pair"] * pairs / t_sample / 1e12 / alu_peak if t_sample else None
            if sc.get("ncu"):
                sample["ncu"] = dict(sc["ncu"], source=sc.get("source"))
        else:
            sample["traffic"] = None
        kernels["compact_kernel"] = compact
        kernels["sample_kernel"] = sample
        dom = sample if t_sample >= t_compact else compact
    roof = dict(dom)
    roof["peak_note"] = peak_src if roof.get("unit") == "GB/s" else roof.get("peak_source")
    roof["kernels"] = dict(kernels, redo_ms=t_redo * 1e3,
                           gather_and_measures_ms=sum(a.elapsed_time(b) for a, b in meas_ev) / max(len(meas_ev), 1))
    roof["path_hbm"] = {"alg_bytes_per_step": alg_bytes, "step_ms": step_s * 1e3,
                        "achieved": alg_bytes / step_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": alg_bytes / step_s / 1e9 / hbm_peak}
    if not primary:
        t_floor = max(alg_bytes / hbm_peak / 1e9, ALG_INST_PER_SAMPLE * pairs / alu_peak / 1e12)
        roof["path_binding"] = {"floor_ms": t_floor * 1e3, "frac": t_floor / step_s,
                                "rule": "max(algorithmic bytes / HBM peak, 300 lane-instructions per SU "
                                        "sample / ALU peak) over the step time (SURVEY 8(d))"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        n = oracle_sample_size(cfg, cores)
        dt, n = time_oracle(cfg, n, cores)
        n1 = max(200, min(10000, oracle_sample_size(cfg, 1, target_s=6.0)))
        dt1, n1 = time_oracle(cfg, n1, 1)
        cpu = {"value": n / dt, "unit": "trials/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"first {n} trials of {cfg['name']} (global index 0..{n - 1}), "
                         f"fp64 C oracle, {cores} threads, {dt:.1f} s",
               "single_core": {"value": n1 / dt1, "unit": "trials/s", "cores": 1,
                               "sample": f"first {n1} trials, 1 thread, {dt1:.1f} s"}}

    n_batches = int(kern_ms[-1].get("batches", 1)) if kern_ms else 1
    # libara kernels per timed step: ara_run's (counted by the library) + one joint-select
    # launch per measured table
    n_meas = len(table_shard(len(layers), rank, world)) if world > 1 and len(layers) > 1 else len(layers)
    gpu_launches = sum(k["launches"] for k in kern_ms) + args.steps * n_meas   # (this rank's selects)
    ms = elapsed / args.steps * 1e3
    value = N_total / (elapsed / args.steps)
    line = {
        "metric": "ARA trials/s", "value": value, "unit": "trials/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg), "n_trials_total": N_total,
                   "trials_per_rank": n_loc, "return_periods": rps,
                   "l2": "inputs > L2: the YET (4 B x events) is streamed every step; the portfolio "
                         "tables (index, bitmap, records) stay L2-resident by design",
                   "parallelism": f"trial-sharded x{world}" + (f" + {backend.upper()} YLT all-gather" if world > 1 else ""),
                   "path": "primary (no draws): one streaming kernel" if primary else
                           f"compaction + sampler, {n_batches} trial batch(es)",
                   "launch": "CUDA graph: one captured step (ara_run ARA_ASYNC + ara_risk_measures_async) "
                             "replayed per timed step" if graph is not None else "eager launches"},
        "e2e": e2e_main,
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torch.distributed.run
        import subprocess
        cmd = launch_command(args.gpus, sys.argv[1:])
        r = subprocess.run(cmd)
        sys.exit(r.returncode)
    rank, world, local = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; run with --gpus equal to the rank count")
    name = args.config or "cfg3"
    if name.endswith(".json"):                 # (a config file: test shapes of the multi-rank path)
        with open(name) as f:
            cfg = aragen.load_config(json.load(f))
    else:
        cfg = aragen.load_config(name)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
    else:
        run_ours(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
