#!/usr/bin/env python
"""Benchmark of the B200 sequence-criterion hot path (BASELINE.json metric:
"ASG/CTC loss+grad frames/sec (B x T) at 1/2/4/8 B200; % of HBM/SFU roofline").

One step = batched ASG loss+grad (fcc - fac, grads w.r.t. emissions and
transitions, transition-gradient all-reduce across ranks) AND batched CTC
loss+grad on the same log-softmaxed emissions, for a
per-GPU shard of B=64 utterances, T=1600 frames, N=30 tokens, L=300 labels
(the C3 shape; at 8 GPUs the global batch is C5's B=512 -> weak scaling).
ASG and CTC run concurrently on two streams.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--global-batch G]   # strong scaling: G utterances split over N

Multi-GPU: one process per GPU (torchrun; with --gpus N > 1 and no
WORLD_SIZE in the environment the script re-launches itself under
torch.distributed.run).  Contiguous batch shards (trainer.py:433), ONE
all-reduce of the 3.6 KB transition gradient per step through the library's
own NCCL entry (w2l_allreduce_grad_A) on the compute stream; timing is the
max over ranks.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ASG/CTC loss+grad frames/sec (B×T) at 1/2/4/8 B200; % of HBM/SFU roofline"
B_PER_GPU, T_FR, N_TOK, L_LAB = 64, 1600, 30, 300
SEED = 20260004  # 20260000 + config index (C5)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
# The two-criteria step's schedule (A/B knobs):
# staggered start (W2L_BENCH_STAGGER=0 starts both criteria together), which
# criterion starts first (W2L_BENCH_FIRST=asg|ctc), and which criteria stream
# their gradient behind their chains (W2L_FLAG_STREAM_GRAD)
STAGGER = os.environ.get("W2L_BENCH_STAGGER", "1") != "0"
FIRST = os.environ.get("W2L_BENCH_FIRST", "asg")
STREAM_ASG = os.environ.get("W2L_BENCH_STREAM_ASG", "1") != "0"
STREAM_CTC = os.environ.get("W2L_BENCH_STREAM_CTC", "1") != "0"
# diagnostics only (the bound on what skipping the empty fallback tiers would
# save; a bench line taken with it is not valid: the precision tiers are part
# of the contract)
FB_KW = {"fallback": False} if os.environ.get("W2L_BENCH_NOFB") == "1" else {}
SIDE_PRIO = int(os.environ.get("W2L_BENCH_SIDE_PRIO", "0"))   # second stream's priority (A/B)


# ---------------------------------------------------------------- inputs --

def make_inputs(rank: int, b=B_PER_GPU, t=T_FR, n=N_TOK, l=L_LAB):
    """Seeded synthetic block `rank` of 64 utterances: emissions
    log_softmax(2 N(0,1)) (f64 -> f32; valid CTC input, used for ASG too),
    ASG targets without consecutive duplicates, CTC targets over the N-1
    non-blank ids, N(0,1) transitions (identical on every rank)."""
    rng = np.random.default_rng(SEED + 1000 * rank)
    x = 2.0 * rng.standard_normal((b, t, n))
    x -= x.max(axis=2, keepdims=True)
    em = (x - np.log(np.exp(x).sum(axis=2, keepdims=True))).astype(np.float32)
    asg_t = np.empty((b, l), np.int64)
    for i in range(b):
        row = rng.integers(0, n - 1, size=l)
        for k in range(1, l):                       # no consecutive duplicates
            if row[k] == row[k - 1]:
                row[k] = (row[k] + 1) % n
        asg_t[i] = row
    ctc_t = rng.integers(0, n - 1, size=(b, l)).astype(np.int64)
    trans = np.random.default_rng(SEED).standard_normal((n, n)).astype(np.float32)
    em_len = np.full(b, t, np.int32)
    tgt_len = np.full(b, l, np.int32)
    return em, em_len, asg_t, ctc_t, tgt_len, trans, n - 1


def shard_inputs(lo: int, hi: int):
    """Utterances [lo, hi) of the global synthetic batch (utterance u lives in
    block u // 64 of make_inputs), so every rank generates only its shard."""
    parts = []
    for blk in range(lo // B_PER_GPU, (hi - 1) // B_PER_GPU + 1):
        em, el, ta, tc, tl, trans, blank = make_inputs(blk)
        a, z = max(lo - blk * B_PER_GPU, 0), min(hi - blk * B_PER_GPU, B_PER_GPU)
        parts.append((em[a:z], el[a:z], ta[a:z], tc[a:z], tl[a:z]))
    cat = [np.concatenate([p[k] for p in parts]) for k in range(5)]
    return (*cat, trans, blank)


def peaky_inputs(scale: float, b=B_PER_GPU, t=T_FR, n=N_TOK, l=L_LAB):
    """The bench shape with log_softmax(scale N(0,1)) emissions (trained
    acoustic models are peaky); targets and transitions as make_inputs(0)."""
    em, el, ta, tc, tl, trans, blank = make_inputs(0, b, t, n, l)
    rng = np.random.default_rng(SEED + 7)
    x = scale * rng.standard_normal((b, t, n))
    x -= x.max(axis=2, keepdims=True)
    em = (x - np.log(np.exp(x).sum(axis=2, keepdims=True))).astype(np.float32)
    return em, el, ta, tc, tl, trans, blank


# ----------------------------------------------------------- CPU baseline --
# The reference's own functions (asrkit.criterion, installed unmodified into
# baseline/_ref) when present -- kind "reference" -- else the oracle port
# (oracle/criterion_oracle.py, the same algorithm restated) -- kind "port".

def _ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "asrkit"))


def _cpu_impl():
    if _ref_available():
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from asrkit import criterion as rc
        return (lambda e, y, a: rc.asg_loss_grad(e, y, a),
                lambda e, y, blank: rc.ctc_loss_grad(e, y, blank), "reference")
    from oracle import criterion_oracle as orc
    return orc.asg, orc.ctc, "port"


def _cpu_worker(args):
    asg, ctc, _ = _cpu_impl()
    e, ya, yc, a, blank = args
    asg(e, ya, a)
    ctc(e, yc, blank)
    return e.shape[0]


def _pool(cores):
    import concurrent.futures as cf
    import multiprocessing as mpc
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    pool = cf.ProcessPoolExecutor(max_workers=cores, mp_context=mpc.get_context("fork"))
    pool.submit(os.getpid).result()   # fork every worker now, before CUDA initialises
    return pool


def _tasks(inp, n_utts):
    em, _, asg_t, ctc_t, _, trans, blank = inp
    return [(em[i % len(em)], asg_t[i % len(em)], ctc_t[i % len(em)], trans, blank)
            for i in range(n_utts)]


def cpu_rates(pool, cores, inp, steps, warmup, min_s=8.0):
    """Frames/s of the CPU implementation on this host: the process pool
    (one utterance per task, all cores: the strongest honest CPU baseline),
    warmed and timed exactly like the reference arm; plus the single-core
    rate and the reference trainer's as-shipped thread pool
    (trainer.py:424-437, GIL-bound)."""
    n_utts = max(16, min(cores, 64))
    tasks = _tasks(inp, n_utts)
    for _ in range(warmup):
        sum(pool.map(_cpu_worker, tasks))
    # at least `steps` passes and min_s seconds (the hosts are shared: a
    # sub-second sample varied by +-20% between back-to-back runs)
    frames, passes, t0 = 0, 0, time.perf_counter()
    while passes < steps or time.perf_counter() - t0 < min_s:
        frames += sum(pool.map(_cpu_worker, tasks))
        passes += 1
    proc_fps = frames / (time.perf_counter() - t0)
    _cpu_worker(tasks[0])
    t0 = time.perf_counter()
    single_fps = _cpu_worker(tasks[0]) / (time.perf_counter() - t0)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=cores) as tp:
        t0 = time.perf_counter()
        thread_fps = sum(tp.map(_cpu_worker, tasks[:cores])) / (time.perf_counter() - t0)
    return proc_fps, single_fps, thread_fps, n_utts, passes


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during timing."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------- roofline --

def algorithmic_work(n=N_TOK, l=L_LAB, ctc_targets=None):
    """Per-frame algorithmic work of the reference algorithm:
    log-semiring transcendental ops (the SFU bound of the log-space
    recursions) and HBM bytes (emissions in, gradient out)."""
    s = 2 * l + 1
    if ctc_targets is not None:
        k = float(np.mean(np.sum(ctc_targets[:, 1:] != ctc_targets[:, :-1], axis=1)))
    else:
        k = (l - 1) * (n - 2) / (n - 1)
    asg_chain = 2 * (n * n + n) + 4 * (l - 1)          # fcc alpha/beta + fac alpha/beta
    asg_grad = (n * n + n) + (l + 2 * l - 1)           # full node+edge, con node+edges
    ctc_chain = 4 * (s - 1 + k)                        # alpha/beta, 2 per logadd edge
    ctc_grad = s + n + 1                               # posteriors + row check
    return {"asg_chain": asg_chain, "asg_grad": asg_grad, "ctc_chain": ctc_chain,
            "ctc_grad": ctc_grad, "bytes_asg": 8 * n, "bytes_ctc": 8 * n}


def _ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------- launcher --

def _relaunch(args):
    """--gpus N > 1 without torchrun: re-exec under torch.distributed.run,
    one process per GPU (the driver launches torchrun itself)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------- main --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling: this many utterances split over the ranks "
                         "(default: weak scaling, 64 per GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-benchmarks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, world, rank)

    # CPU baseline (rank 0 at N=1 only), timed before CUDA initialises: run
    # after the GPU phase, the same pool measured ~1.5x below the reference
    # arm's fresh process on the same box
    cores = cpu_cores()
    cpu_meas = None
    if world == 1 and not args.no_cpu_baseline:
        with _pool(cores) as pool:
            cpu_meas = cpu_rates(pool, cores, make_inputs(0), 3, 3)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1812_07625_b200 import _native, criterion as C
    from paper_1812_07625_b200.distributed import NcclComm, shard_bounds

    strong = args.global_batch is not None
    g_batch = args.global_batch if strong else world * B_PER_GPU
    lo, hi = shard_bounds(g_batch, world, rank)
    em, em_len, asg_t, ctc_t, tgt_len, trans, blank = shard_inputs(lo, hi)
    B, T, N = em.shape
    comm = NcclComm() if world > 1 else None
    em_d = torch.from_numpy(em).to(dev)
    el_d = torch.from_numpy(em_len).to(dev)
    ta_d = torch.from_numpy(asg_t).to(dev)
    tc_d = torch.from_numpy(ctc_t).to(dev)
    tl_d = torch.from_numpy(tgt_len).to(dev)
    A_d = torch.from_numpy(trans).to(dev)
    lib = _native.lib()
    ws_a = torch.empty(lib.w2l_asg_workspace_bytes(B, T, N, L_LAB), dtype=torch.uint8, device=dev)
    ws_c = torch.empty(lib.w2l_ctc_workspace_bytes(B, T, N, L_LAB), dtype=torch.uint8, device=dev)
    out_a = C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=True, workspace=ws_a)
    out_c = C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=True, workspace=ws_c)
    # the fp32 path must not have needed the float64 fallback on this data
    chk_a = C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                    fallback=False)
    chk_c = C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c,
                                    fallback=False)
    fallbacks = int((chk_a.status != 0).sum().item() + (chk_c.status != 0).sum().item())

    side = torch.cuda.Stream(device=dev, priority=SIDE_PRIO)
    main_s = torch.cuda.current_stream(dev)
    validated = torch.cuda.Event()   # the first criterion's validation done (staggered start)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def both(em_, el_, ta_, tc_, tl_, outs=None):
        oa_, oc_ = outs if outs is not None else (out_a, out_c)

        def asg(**kw):
            return C.asg_loss_grad_batched(em_, el_, ta_, tl_, A_d, check=False, workspace=ws_a,
                                           out=oa_, stream_grad=STREAM_ASG, **kw, **FB_KW)

        def ctc(**kw):
            return C.ctc_loss_grad_batched(em_, el_, tc_, tl_, blank, check=False, workspace=ws_c,
                                           out=oc_, stream_grad=STREAM_CTC, **kw, **FB_KW)

        # The two criteria run concurrently on two streams (the chain CTAs of
        # both are co-resident: maximum shared-memory carveout).  Staggered
        # start: the second criterion begins its validation when the first's
        # has finished, so its recursions start ~20 us later.  Started
        # together, the two chains sharing each SM fall into a slow mode on
        # about two thirds of the steps (per-step device times 0.49 vs
        # 0.53-0.58 ms, tools/step_times.py).  ASG (the longer chains) goes
        # first.  Both stream their gradients behind their chains (CTC's too
        # since the ASG gradient runs 4 CTAs per SM: device step -2..-4%,
        # e2e equal, 8 A/B pairs on two boxes).
        first, second = (asg, ctc) if FIRST == "asg" else (ctc, asg)
        side.wait_stream(main_s)
        if STAGGER:
            o1 = first(phase="validate")
            validated.record(main_s)
            o1 = first(phase="rest")
            side.wait_event(validated)
        else:
            o1 = first()
        with torch.cuda.stream(side):
            o2 = second()
        oa, oc = (o1, o2) if FIRST == "asg" else (o2, o1)
        if comm is not None:      # the one exchange: sum of grad_A over ranks
            comm.allreduce_grad_transitions(oa.grad_transitions)
        main_s.wait_stream(side)
        return oa, oc

    def step():
        both(em_d, el_d, ta_d, tc_d, tl_d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()                      # evict L2 between timed steps
            starts[i].record(main_s)
            step()
            ends[i].record(main_s)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    frames_step = g_batch * T
    value = frames_step * args.steps / (total_ms / 1e3)

    # ---- end to end through the public API: pinned host inputs -> device ->
    # both criteria -> losses back to the host, every step (and a variant that
    # also returns both gradients to the host, as the reference API does)
    em_h = torch.from_numpy(em).pin_memory()
    ta_h = torch.from_numpy(asg_t).pin_memory()
    tc_h = torch.from_numpy(ctc_t).pin_memory()
    el_h = torch.from_numpy(em_len).pin_memory()
    tl_h = torch.from_numpy(tgt_len).pin_memory()
    loss_a_h = torch.empty(B, dtype=torch.float64).pin_memory()
    loss_c_h = torch.empty(B, dtype=torch.float64).pin_memory()
    ge_a_h = torch.empty((B, T, N), dtype=torch.float32).pin_memory()
    ge_c_h = torch.empty((B, T, N), dtype=torch.float32).pin_memory()
    ga_h = torch.empty((N, N), dtype=torch.float32).pin_memory()
    # double-buffered device inputs: a copy stream brings step i+1's inputs in
    # while step i computes (each step still copies its own inputs and reads
    # its results back; only the overlap is new)
    bufs = [dict(em=torch.empty_like(em_d), ta=torch.empty_like(ta_d), tc=torch.empty_like(tc_d),
                 el=torch.empty_like(el_d), tl=torch.empty_like(tl_d)) for _ in range(2)]
    copy_s = torch.cuda.Stream(device=dev)
    d2h_s = torch.cuda.Stream(device=dev)   # read-back off the compute stream
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    read_back = [torch.cuda.Event() for _ in range(2)]
    outs = [(out_a, out_c),
            (C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a),
             C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                     workspace=ws_c))]

    def e2e_step(i, grads):
        bi = bufs[i & 1]
        with torch.cuda.stream(copy_s):
            if i >= 2:
                copy_s.wait_event(consumed[i & 1])     # buffer free again
            bi["em"].copy_(em_h, non_blocking=True)
            bi["ta"].copy_(ta_h, non_blocking=True)
            bi["tc"].copy_(tc_h, non_blocking=True)
            bi["el"].copy_(el_h, non_blocking=True)
            bi["tl"].copy_(tl_h, non_blocking=True)
            copied[i & 1].record(copy_s)
        main_s.wait_event(copied[i & 1])
        if i >= 2:
            main_s.wait_event(read_back[i & 1])       # outputs free again
        # (the CTC stream waits for everything on main: letting a step's CTC
        # chain start under the previous step's ASG gradient measured slower,
        # 1.80-1.87e8 vs 1.89-1.91e8 frames/s)
        oa, oc = both(bi["em"], bi["el"], bi["ta"], bi["tc"], bi["tl"], outs[i & 1])
        consumed[i & 1].record(main_s)
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_event(consumed[i & 1])
            loss_a_h.copy_(oa.loss, non_blocking=True)
            loss_c_h.copy_(oc.loss, non_blocking=True)
            if grads:
                ge_a_h.copy_(oa.grad_emissions, non_blocking=True)
                ge_c_h.copy_(oc.grad_emissions, non_blocking=True)
                ga_h.copy_(oa.grad_transitions, non_blocking=True)
            read_back[i & 1].record(d2h_s)

    def e2e_run(grads):
        for i in range(args.warmup):
            e2e_step(i, grads)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        # steps are queued back to back; the clock starts before the first
        # input copy and stops after the last results reached the host
        e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        torch.cuda.synchronize(dev)
        e_s.record(main_s)
        copy_s.wait_stream(main_s)
        h0 = time.perf_counter()
        for i in range(args.steps):
            e2e_step(i, grads)
        host_ms.append((time.perf_counter() - h0) * 1e3 / args.steps)
        main_s.wait_stream(d2h_s)
        e_e.record(main_s)
        e_e.synchronize()
        t = torch.tensor([e_s.elapsed_time(e_e)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return frames_step * args.steps / (float(t.item()) / 1e3)

    host_ms = []   # host enqueue time per e2e step (is the e2e host-bound?)
    e2e_value = e2e_run(False)
    e2e_grads_value = e2e_run(True)
    h2d = em.nbytes + asg_t.nbytes + ctc_t.nbytes + em_len.nbytes + tgt_len.nbytes
    d2h = 2 * B * 8
    d2h_grads = d2h + 2 * em.nbytes + N * N * 4

    if world > 1:
        dist.barrier()
    if rank != 0:
        comm.close()
        dist.destroy_process_group()
        return

    # ---- per-stage device times (traced calls) and the roofline of the
    # dominant kernel; sub-benchmarks per criterion, Viterbi and peaky inputs
    torch.cuda.synchronize(dev)
    ta_run = C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                     trace=True)
    tc_run = C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                     workspace=ws_c, trace=True)
    peaks = _native.probe_peaks()
    work = algorithmic_work(ctc_targets=ctc_t)
    frames = B * T
    stages = {("asg", k): v for k, v in ta_run.stage_ms.items()}
    stages.update({("ctc", k): v for k, v in tc_run.stage_ms.items()})
    (crit, stage), dom_ms = max(stages.items(), key=lambda kv: kv[1])
    ops_key = f"{crit}_{stage}" if f"{crit}_{stage}" in work else None
    sfu_ops = work[ops_key] * frames if ops_key else None
    roof_sfu = {
        "kernel": f"{crit}_{stage}",
        "bound": "sfu",
        "achieved": (sfu_ops / (dom_ms / 1e3) / 1e9) if sfu_ops else None,
        "peak": peaks["mufu_ex2_per_s"] / 1e9,
        "unit": "Gop/s (log-semiring transcendental ops, SURVEY §8d)",
        "frac": (sfu_ops / (dom_ms / 1e3) / peaks["mufu_ex2_per_s"]) if sfu_ops else None,
        "kernel_ms": dom_ms,
        "peak_source": "w2l_probe_peaks: MUFU ex2 throughput measured on this GPU",
    }
    hbm_peak, hbm_src = _hbm_peak()
    step_s = total_ms / args.steps / 1e3
    step_bytes = (work["bytes_asg"] + work["bytes_ctc"]) * frames
    step_ops = (work["asg_chain"] + work["asg_grad"] + work["ctc_chain"] + work["ctc_grad"]) * frames
    # HBM roofline of the dominant stage: its algorithmic bytes per launch
    # (chain = emissions in, 4N B/frame; gradient = emissions in +
    # gradient out, 8N B/frame; workspace rows are implementation traffic)
    dom_alg_bytes = (4 if stage == "chain" else 8) * N * frames
    roof = {
        "kernel": f"{crit}_{stage}",
        "bound": "hbm",
        "achieved": dom_alg_bytes / (dom_ms / 1e3) / 1e9,
        "peak": hbm_peak,
        "unit": "GB/s",
        "frac": dom_alg_bytes / (dom_ms / 1e3) / 1e9 / hbm_peak,
        "traffic": _ncu_traffic(f"{crit}_{stage}"),
        "alg_bytes_per_launch": dom_alg_bytes,
        "kernel_ms": dom_ms,
        "peak_source": hbm_src,
        "note": ("serial T-step recursion: latency-bound; the SFU-equivalent view is in "
                 "roofline_sfu, the latency view in roofline_latency") if stage == "chain" else
                ("posterior/gradient kernels: achieved counts only the algorithmic bytes "
                 "(emissions in, gradient out); traffic adds the workspace it reads"),
        "step": {
            "sfu_ops_per_step": step_ops,
            "sfu_achieved_gops": step_ops / step_s / 1e9,
            "sfu_frac": step_ops / step_s / peaks["mufu_ex2_per_s"],
            "hbm_bytes_per_step": step_bytes,
            "hbm_achieved_gbs": step_bytes / step_s / 1e9,
            "hbm_peak_gbs": hbm_peak,
            "hbm_frac": step_bytes / step_s / 1e9 / hbm_peak,
        },
    }
    # latency roofline of the serial recursions: T dependent steps, each at
    # least the measured one-warp step floor (fcc ~174 cycles,
    # lattice ~30 cycles of recursion arithmetic), at the sampled SM clock
    clk_sum = clk.summary()
    mhz = clk_sum.get("sm_mhz") or 1965.0
    chain_ms = {c: stages.get((c, "chain")) for c in ("asg", "ctc")}
    floor_cycles = {"asg": 174, "ctc": 30}
    roof_lat = {c: {"kernel_ms": chain_ms[c], "floor_cycles_per_step": floor_cycles[c],
                    "floor_ms": T * floor_cycles[c] / (mhz * 1e3),
                    "cycles_per_step": (chain_ms[c] * mhz * 1e3 / T) if chain_ms[c] else None,
                    "frac": (T * floor_cycles[c] / (mhz * 1e3) / chain_ms[c]) if chain_ms[c] else None}
                for c in ("asg", "ctc")}

    roof_dram = {}
    for crit_, stages_ in (("asg", ta_run.stage_ms), ("ctc", tc_run.stage_ms)):
        traffic = _ncu_traffic(f"{crit_}_grad")
        if traffic and stages_.get("grad"):
            gbs = traffic / (stages_["grad"] / 1e3) / 1e9
            roof_dram[f"{crit_}_grad"] = {"dram_bytes_per_launch": traffic,
                                         "kernel_ms": stages_["grad"], "achieved_gbs": gbs,
                                         "frac": gbs / hbm_peak}
    roof_dram = {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "peak_source": hbm_src,
                 "kernels": roof_dram} if roof_dram else None

    sub = {"asg_stage_ms": ta_run.stage_ms, "ctc_stage_ms": tc_run.stage_ms,
           "peaks": peaks, "fp32_guard_fallbacks": fallbacks}
    roof_vit = None
    if not args.no_sub:
        def timeit(fn, reps=5):
            fn()
            torch.cuda.synchronize(dev)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot = 0.0
            for _ in range(reps):
                flush.zero_()
                s_.record()
                fn()
                e_.record()
                e_.synchronize()
                tot += s_.elapsed_time(e_)
            return tot / reps
        ms_a = timeit(lambda: C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False,
                                                      workspace=ws_a, out=out_a))
        ms_c = timeit(lambda: C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank,
                                                      check=False, workspace=ws_c, out=out_c))
        ms_v = timeit(lambda: C.viterbi_batched(em_d, el_d, A_d, check=False))
        ms_al = timeit(lambda: C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False,
                                                       workspace=ws_a, out=out_a, loss_only=True))
        ms_cl = timeit(lambda: C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank,
                                                       check=False, workspace=ws_c, out=out_c,
                                                       loss_only=True))
        ms_cx = timeit(lambda: C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank,
                                                       check=False, workspace=ws_c, out=out_c,
                                                       logits=True))
        sub.update({"asg_only_frames_per_s": frames / (ms_a / 1e3), "asg_only_ms": ms_a,
                    "ctc_only_frames_per_s": frames / (ms_c / 1e3), "ctc_only_ms": ms_c,
                    "viterbi_frames_per_s": frames / (ms_v / 1e3), "viterbi_ms": ms_v,
                    "asg_loss_only_ms": ms_al, "ctc_loss_only_ms": ms_cl,
                    "ctc_logits_fused_ms": ms_cx})
        # Viterbi against its own bound: 2N^2 + N float64 add/compare ops per
        # frame over the measured DADD rate
        vit_ops = (2 * N * N + N) * frames
        roof_vit = {"kernel": "viterbi", "bound": "fp64", "unit": "Gop/s",
                    "achieved": vit_ops / (ms_v / 1e3) / 1e9,
                    "peak": peaks["dadd_per_s"] / 1e9,
                    "frac": vit_ops / (ms_v / 1e3) / peaks["dadd_per_s"], "kernel_ms": ms_v,
                    "peak_source": "w2l_probe_peaks: DADD throughput measured on this GPU"}
        # peaky emissions (trained models): fp32-guard failures, and the step
        # time with the precision routing (default: a batch the fp32 tier
        # would fail goes straight to the fp64 tier) and without it (fp32
        # pass, then the fp64 tier for its failures)
        peaky = {}
        for scale in (2.0, 5.0, 10.0, 20.0):
            pe = peaky_inputs(scale, b=B)
            pem = torch.from_numpy(pe[0]).to(dev)
            pa = C.asg_loss_grad_batched(pem, el_d, ta_d, tl_d, A_d, check=False,
                                         workspace=ws_a, fallback=False)
            pc = C.ctc_loss_grad_batched(pem, el_d, tc_d, tl_d, blank, check=False,
                                         workspace=ws_c, fallback=False)
            fa, fc = int((pa.status != 0).sum().item()), int((pc.status != 0).sum().item())
            row = {"asg_fallbacks": fa, "ctc_fallbacks": fc}
            for tag, rt in (("", True), ("_unrouted", False)):
                row["asg_ms" + tag] = timeit(lambda: C.asg_loss_grad_batched(
                    pem, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, route=rt), reps=2)
                row["ctc_ms" + tag] = timeit(lambda: C.ctc_loss_grad_batched(
                    pem, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, route=rt),
                    reps=2)
            row["asg_vs_fast"] = row["asg_ms"] / ms_a
            row["ctc_vs_fast"] = row["ctc_ms"] / ms_c
            peaky[f"s={scale:g}"] = row
        sub["peaky_emissions"] = peaky

    cpu = None
    if cpu_meas is not None:
        proc_fps, single_fps, thread_fps, n_utts, passes = cpu_meas
        kind = "reference" if _ref_available() else "port"
        cpu = {"value": proc_fps, "unit": "frames/s", "cores": cores, "kind": kind,
               "cpu": cpu_model(),
               "single_core_frames_per_s": single_fps,
               "thread_pool_frames_per_s": thread_fps,
               "sample": f"{n_utts} utterances (T={T}, N={N}, L={L_LAB}) ASG+CTC loss+grad, "
                         + ("asrkit.criterion (the reference, baseline/_ref)" if kind == "reference"
                            else "oracle port (float64 numpy)")
                         + f", one utterance per task, process pool of {cores} (3 warm-up + {passes} "
                           "timed passes, >= 8 s, before the GPU phase); "
                           "single core: 1 utterance; thread pool (trainer.py:424-437): "
                           f"{cores} utterances on {cores} threads"}

    # our kernels per step: ASG em_check, prep, chain, grad, final, exact
    # (fallback, early exit), reduce; CTC em_check, prep, chain, grad, final,
    # exact (+ the NCCL all-reduce at N > 1)
    # library kernels per step (the ncu launch list, profiles/r2): ASG em_check,
    # prep, chain, grad, final, fp64 chain / grad / final, log-domain, reduce
    # (10); CTC the same without the reduction (9).  The status and routing
    # memsets are not counted.
    launches_per_step = 10 + 9
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic seeded: log_softmax(2*N(0,1)) emissions, N(0,1) transitions, "
                "uniform targets",
        "config": {"workload": f"ASG+CTC loss+grad, B={B}/GPU T={T} N={N} L={L_LAB} "
                               + ("(strong scaling)" if strong else
                                  "(C3 shape per GPU; C5 B=512 at 8 GPUs)"),
                   "global_batch": g_batch, "frames_per_step": frames_step,
                   "parallelism": f"dp{world}", "l2": "flushed (256 MiB write) between steps",
                   "schedule": (f"two streams, {FIRST} first"
                                + (", staggered" if STAGGER else ", together")
                                + "; streamed gradient: "
                                + ("+".join([k for k, v in (("asg", STREAM_ASG),
                                                            ("ctc", STREAM_CTC)) if v])
                                   or "none"))},
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "boundary": "pinned host inputs in, per-utterance losses out (on-GPU training "
                            "keeps the gradients on the device)",
                "host_enqueue_ms_per_step": round(host_ms[0], 4)},
        "e2e_grads_to_host": {"value": e2e_grads_value, "unit": "frames/s",
                              "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h_grads,
                              "boundary": "as e2e, plus both emission gradients and grad_A "
                                          "back to pinned host memory (the reference API's "
                                          "return values)",
                              "host_enqueue_ms_per_step": round(host_ms[1], 4)},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "roofline_sfu": roof_sfu,
        "roofline_latency": roof_lat,
        "roofline_viterbi": roof_vit,
        "roofline_dram_grad": roof_dram,
        "cpu_baseline": cpu,
        "clocks": clk_sum,
        "sub": sub,
        "library": lib.w2l_version().decode(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        comm.close()
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """The reference's CPU implementation of the path on this host's cores:
    asrkit.criterion's asg_loss_grad + ctc_loss_grad (installed unmodified in
    baseline/_ref) when present, else the oracle port; one utterance per task
    in a process pool over every core; rank 0 only."""
    if rank != 0:
        return
    inp = make_inputs(0)
    cores = cpu_cores()
    kind = "reference" if _ref_available() else "port"
    with _pool(cores) as pool:
        n_utts = max(16, min(cores, 64))
        tasks = _tasks(inp, n_utts)
        for _ in range(args.warmup):
            sum(pool.map(_cpu_worker, tasks))
        frames = 0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            frames += sum(pool.map(_cpu_worker, tasks))
        total = time.perf_counter() - t0
    value = frames / total
    impl = ("asrkit.criterion.asg_loss_grad + ctc_loss_grad (the reference, baseline/_ref)"
            if kind == "reference" else "oracle port (float64 numpy)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic seeded (same generator as the GPU arm)",
        "config": {"workload": f"ASG+CTC loss+grad, T={T_FR} N={N_TOK} L={L_LAB}; each step a "
                               f"{n_utts}-utterance sample of the B={B_PER_GPU} shard",
                   "global_batch": n_utts, "parallelism": f"process pool x{cores}"},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": kind,
                         "cpu": cpu_model(), "impl": impl,
                         "sample": f"{n_utts} utterances per step, one per task"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
