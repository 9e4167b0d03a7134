#!/usr/bin/env python
"""Benchmark of the Nimbus COP hot path (Alg. 1 steps 2-4)
on B200: one `step` = one pass of the client's COP matmuls (slice X -> tcgen05
contraction -> RShift packing + mod-switch + mask) over one batch of synthetic
inputs with Enc(W) resident in HBM.

Default line = BASELINE.json configs[4] (C5): the full BERT-base linear stack,
12 layers x (Q, K, V, O 768x768, FFN-up 768x3072, FFN-down 3072x768) = 72
matmuls of k = 2048 rows (seq 512 x 4 queries), N=8192, 3 limbs, ell=32 -- the
north star's "BERT-base FFN layers" in their full-model setting.  The same line
carries `per_config`: C2 (attention projection), C3 (FFN up), C4 (FFN down),
each with its own ms_per_step, roofline, cpu_baseline and e2e, plus C4 and C5 at
ell = 16 (SURVEY.md 8(c) #2's secondary line) and the paper's ell = 64 (C4@l64,
C5@l64) as secondary entries.  `--config K` times one config
alone (1..5; 4l16 / 5l16 / 4l64 / 5l64 the secondary parameter sets).

Prints ONE JSON line (rank 0).  Multi-GPU (torchrun): every rank runs its own
independent queries against its own copy of Enc(W) (weak scaling, no
data-path collective); timing is the max over ranks.

--impl reference runs the CPU oracle (oracle/, the reference arm of this
tier) on the same config, each step a bounded row sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import nimbus_inputs as ni  # noqa: E402

METRIC = "COP matmul ms/layer and modular MAC/s (BERT-base shapes) vs int8 TC roofline"
UNIT = "modMAC/s"
L2_FLUSH_BYTES = 512 << 20     # > 126 MB L2, written between timed steps


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, help="one config alone (default: C5 with per_config entries)")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false")
    ap.add_argument("--impl", default="tcgen05", choices=["tcgen05", "cudacore", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profiler-range", action="store_true",
                    help="cudaProfilerStart/Stop around the K block-timed steps (ncu --replay-mode range)")
    ap.add_argument("--prefetch-next", type=int, default=1, choices=[0, 1, 2],
                    help="k = 128 configs: hint the next step's Enc(W) to the library (nimbus_cop_prefetch_next)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="skip the secondary timing of the steps replayed from a CUDA graph")
    ap.add_argument("--cpu-budget-s", type=float, default=8.0,
                    help="oracle seconds per cpu_baseline leg (all cores, then one thread)")
    ap.add_argument("--no-stage-profile", action="store_true", help="no per-stage events inside the step")
    ap.add_argument("--l2", default="rotate", choices=["rotate", "write"],
                    help="cold-L2 method: rotate through input copies totalling >= 3x L2 (default), "
                         "or write a 512 MiB buffer before every timed step")
    return ap.parse_args()


def step_dist(step_ms):
    """median and p10 / p90 of the per-step times (nearest-rank percentiles)."""
    v = sorted(step_ms)
    if not v:
        return None
    pick = lambda q: v[min(len(v) - 1, max(0, int(round(q * (len(v) - 1)))))]
    return {"runs": len(v), "median": statistics.median(v), "p10": pick(0.10), "p90": pick(0.90)}


def get_config(key: str):
    if ":" in key:
        # diagnostic subset of a stack: "5:down" = C5's FFN-down matmuls only (projections Q K V O up down)
        import dataclasses
        base, projs = key.split(":")
        cfg = get_config(base)
        keep = [ni._PROJ.index(p) for p in projs.split(",")]
        return dataclasses.replace(cfg, name=f"{cfg.name}:{projs}",
                                   layers=tuple(x for x in cfg.layers if x[1] in keep))
    if key == "2qkv":
        return ni.CONFIG_QKV
    if key.endswith("l16"):
        return ni.CONFIGS_L16[int(key[0])]
    if key.endswith("l64"):
        return ni.CONFIGS_L64[int(key[0])]
    return ni.CONFIGS[int(key)]


def workload_name(cfg):
    lays = [l for _, _, l in cfg.layers]
    if len(lays) == 1:
        l = lays[0]
        return (f"{cfg.name} {l.name}: X {l.k}x{l.m} . W {l.m}x{l.n}, N={cfg.N}, L={cfg.L}, "
                f"ell={cfg.ell}, L_out={cfg.L_out}")
    if cfg.shared_x:
        l = lays[0]
        return (f"{cfg.name}: {len(lays)} matmuls sharing X ({', '.join(x.name for x in lays)}), each X {l.k}x{l.m} . "
                f"W {l.m}x{l.n}, N={cfg.N}, L={cfg.L}, ell={cfg.ell}, L_out={cfg.L_out}")
    return (f"{cfg.name} BERT-base linear stack: 12 layers x (4x768x768 + 768x3072 + 3072x768), "
            f"k={lays[0].k} (seq {lays[0].k_per_query} x {lays[0].n_queries} queries), N={cfg.N}, "
            f"L={cfg.L}, ell={cfg.ell}, L_out={cfg.L_out}")


def rank_x_seed(seed: int, rank: int) -> int:
    """Weak scaling over independent queries: rank r draws its own client share X."""
    return seed ^ (rank << 40)


def max_over_ranks(x: float, world: int, device) -> float:
    """Max of a per-rank duration over all ranks (torch.distributed, any backend)."""
    if world <= 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def weak_value(macs_per_rank_step: float, world: int, ms_per_step: float) -> float:
    """Whole-job modMAC/s: all ranks' units / the max-over-ranks step time."""
    return macs_per_rank_step * world / (ms_per_step / 1e3)


def sx_of(ell):
    return 1 if ell <= 8 else 2 if ell <= 16 else 4 if ell <= 32 else 8


def measured_peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        p.update({k: d[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in d})
        p["src"] = "MEASURED_PEAKS.json"
    return p


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_samples(self, n, timeout_s=3.0, busy=None):
        """Block until `n` samples in total have arrived (nvidia-smi needs ~0.1-0.3 s to
        start and samples every 100 ms); `busy()` keeps the GPU under the same load."""
        t0 = time.time()
        while self.proc is not None and len(self.lines) < n and time.time() - t0 < timeout_s:
            if busy is not None:
                busy()
            else:
                time.sleep(0.01)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


# ----------------------------------------------------------------- GPU arm
def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    from paper_2411_15707_b200 import nimbus as nb

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    impl = nb.IMPL_TCGEN05 if args.impl == "tcgen05" else nb.IMPL_CUDACORE
    # layout hint: matmuls of >= 512 rows (C5) favour the transposed ell = 32 contraction
    flags = nb.FLAG_LARGE_K if min(l.k for _, _, l in cfg.layers) >= 512 else 0
    ctx = nb.nimbus_ctx_create(cfg.N, cfg.L, cfg.ell, cfg.L_out, impl, flags=flags, device=local_rank)
    sk = nb.nimbus_keygen(ctx, cfg.seed_cfg)
    # setup (untimed, reported separately): encrypt every weight matrix of the workload
    mats = []
    t_setup = 0.0
    enc_bytes = 0
    wide = cfg.ell > 32                      # X, W, R as uint64: the _u64 entry points
    to_dev = nb.from_numpy_u64 if wide else nb.from_numpy_u32
    encrypt = nb.nimbus_encrypt_weights_u64 if wide else nb.nimbus_encrypt_weights
    outputs = nb.alloc_outputs_u64 if wide else nb.alloc_outputs
    matmul = nb.nimbus_cop_matmul_u64 if wide else nb.nimbus_cop_matmul
    for li, pj, lay in cfg.layers:
        seed = ni.seed_mm(cfg.cid, li, pj)
        W = to_dev(ni.gen_W(seed, lay.m, lay.n, cfg.ell), dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        encw = encrypt(ctx, sk, W, seed)
        torch.cuda.synchronize()
        t_setup += time.perf_counter() - t0
        enc_bytes += nb.nimbus_encw_bytes(encw)
        # per-rank independent queries (weak scaling): X seeded by rank; one X for a shared-X step
        xseed = rank_x_seed(seed, rank)
        X = mats[0]["X"][0] if (cfg.shared_x and mats) else to_dev(ni.gen_X(xseed, lay.k, lay.m, cfg.ell), dev)
        cts, R = outputs(ctx, encw, lay.k_per_query, lay.n_queries)
        mats.append(dict(lay=lay, seed=seed, encw=[encw], X=[X], W=W, cts=cts, R=R,
                         ws_bytes=nb.nimbus_cop_workspace_size(ctx, encw, lay.k)))
    # cold L2 without a flush write (whose dirty lines would be written back during
    # the next step): rotate through copies of every input whose total is >= 3x L2,
    # so each step reads Enc(W) and X that were evicted by the steps in between
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    n_copies = 1
    if args.l2 == "rotate":
        n_copies = max(1, -(-3 * l2_bytes // enc_bytes))
        for mt in mats:
            lay = mt["lay"]
            for c in range(n_copies - 1):
                mt["encw"].append(encrypt(ctx, sk, mt["W"], mt["seed"]))
                # a shared-X step keeps one X per copy for all of its matmuls
                mt["X"].append(mats[0]["X"][c + 1] if (cfg.shared_x and mt is not mats[0]) else mt["X"][0].clone())
    # setup on the device, steady state (allocations excluded): re-encrypt the first
    # matrix into its existing handle (nimbus_encrypt_weights_into: the encrypt and tile
    # kernels and a stream-ordered temporary), CUDA events around the stream work
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mt0 = mats[0]
    tmp = encrypt(ctx, sk, mt0["W"], mt0["seed"])       # allocate once
    nb.nimbus_encrypt_weights_into(ctx, sk, mt0["W"], mt0["seed"], tmp)   # warm the temporary pool
    torch.cuda.synchronize()
    t_h0 = time.perf_counter()
    e0.record()
    nb.nimbus_encrypt_weights_into(ctx, sk, mt0["W"], mt0["seed"], tmp)
    e1.record()
    torch.cuda.synchronize()
    setup_host_s = time.perf_counter() - t_h0
    setup_gpu_ms = e0.elapsed_time(e1)
    setup_bytes = nb.nimbus_encw_bytes(tmp)
    del tmp
    for mt in mats:
        del mt["W"]
    torch.cuda.synchronize()
    # one workspace shared by every matmul of the step (they run in stream order)
    ws = torch.empty(max(mt["ws_bytes"] for mt in mats), dtype=torch.uint8, device=dev)
    for mt in mats:
        mt["ws"] = ws
    # multi-matmul steps (C5) go through the batched call: the pack of matmul i
    # overlaps the contraction of matmul i+1 on the library's side stream
    jobs = [[dict(encw=mt["encw"][c], X=mt["X"][c], k_per_query=mt["lay"].k_per_query,
                  n_queries=mt["lay"].n_queries, mask_seed=mt["seed"], cts=mt["cts"], R=mt["R"]) for mt in mats]
            for c in range(n_copies)]
    ws_batch = None
    batch = nb.nimbus_cop_matmul_batch_u64 if wide else nb.nimbus_cop_matmul_batch
    if len(mats) > 1:
        size_fn = nb.nimbus_cop_workspace_size_batch_u64 if wide else nb.nimbus_cop_workspace_size_batch
        ws_batch = torch.empty(size_fn(ctx, jobs[0]), dtype=torch.uint8, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES if args.l2 == "write" else 64 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    step_no = [0]

    def cold():
        """Between timed steps: next input copy (rotate) or an L2 flush write."""
        if args.l2 == "write":
            flush.zero_()
        step_no[0] += 1

    def step_on(st):
        c = step_no[0] % n_copies
        if args.prefetch_next and cfg.ell <= 16 and max(l.k for _, _, l in cfg.layers) <= 128:
            # the model's next matmul (here: the next step's copy) is known: its first Enc(W) tiles
            # are prefetched towards L2 by this step's contraction once its own copies are issued
            # (2: a control -- the hint names a copy that is NOT read next, same prefetch traffic, no hits)
            nxt = (c + 1) % n_copies if args.prefetch_next == 1 else (c + n_copies // 2) % n_copies
            nb.nimbus_cop_prefetch_next(ctx, mats[0]["encw"][nxt])
        if ws_batch is not None:
            batch(ctx, jobs[c], ws_batch, stream=st)
            return
        for mt in mats:
            lay = mt["lay"]
            matmul(ctx, mt["encw"][c], mt["X"][c], lay.k_per_query, lay.n_queries, mt["seed"],
                   mt["cts"], mt["R"], mt["ws"], stream=st)

    def step():
        step_on(stream)

    for _ in range(max(args.warmup, n_copies)):
        cold()
        step()
    torch.cuda.synchronize()
    # clock spin-up outside the workload (memory writes only)
    t0 = time.time()
    while time.time() - t0 < 0.3:
        flush.zero_()
    torch.cuda.synchronize()
    if args.l2 == "rotate":      # leave the L2 holding other copies' inputs, as in steady state
        for _ in range(n_copies):
            cold()
            step()
        torch.cuda.synchronize()

    def timed(profile: bool, per_step: bool):
        """K steps.  per_step: CUDA events around every step (and, with --l2 write, the flush
        between steps outside them); otherwise one event pair around the K back-to-back steps,
        so the PDL chain runs on from one step's pack into the next step's slice and
        contraction (with --l2 rotate every step already reads inputs not in L2)."""
        nb.nimbus_profile_enable(ctx, profile)
        nb.nimbus_profile_read(ctx, reset=True)
        launches0 = nb.nimbus_launch_count(ctx)
        n_ev = args.steps if per_step else 1
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ranged = args.profiler_range and not per_step and not profile
        if ranged:                              # ncu --replay-mode range: the K chained steps as one range
            torch.cuda.profiler.start()
        if not per_step:
            starts[0].record(stream)
        for i in range(args.steps):
            cold()                              # Enc(W), X of this step are not in L2
            if per_step:
                starts[i].record(stream)
            step()
            if per_step:
                ends[i].record(stream)
        if not per_step:
            ends[0].record(stream)
        torch.cuda.synchronize()
        if ranged:
            torch.cuda.profiler.stop()
        if world > 1:
            torch.distributed.barrier()
        launches = nb.nimbus_launch_count(ctx) - launches0
        stage_ms, calls = nb.nimbus_profile_read(ctx, reset=True)
        nb.nimbus_profile_enable(ctx, False)
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total = sum(step_ms)
        total = max_over_ranks(total, world, dev)
        return total, step_ms, stage_ms, calls, launches

    def timed_graph():
        """K steps replayed from a CUDA graph holding n_copies consecutive steps (one per
        input copy, so the rotation is the same as in pass A)."""
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        nonlocal_step = step_no[0]
        with torch.cuda.graph(g, stream=gs, capture_error_mode="thread_local"):
            for c in range(n_copies):
                step_no[0] = c
                step_on(gs)
        step_no[0] = nonlocal_step
        reps = -(-args.steps // n_copies)
        g.replay()
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        a_.record(stream)
        for _ in range(reps):
            g.replay()
        b_.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(a_.elapsed_time(b_), world, dev)
        return ms / (reps * n_copies)

    # pass A (the reported number): the step exactly as a user runs it, no events inside
    # clocks: the sampler is already polling when the timed region starts; a region
    # shorter than its 100 ms period is followed by identical untimed steps until two
    # more samples have landed, so the reported clocks are those of this load
    clocks = ClockSampler(local_rank)
    clocks.start()

    def busy():
        for _ in range(4):
            cold()
            step()
        torch.cuda.synchronize()

    clocks.wait_samples(1, busy=busy)
    n0 = len(clocks.lines)
    total_ms, _, _, _, launches = timed(profile=False, per_step=args.l2 == "write")
    kernel = nb.nimbus_last_contraction(ctx)
    clocks.wait_samples(n0 + 2, busy=busy)
    clk = clocks.stop()
    # pass B (roofline evidence): same K steps with CUDA events around each kernel of the
    # step on its stream; the events serialise the PDL-overlapped launches, so the step
    # is slower here, but each bracketed kernel's own duration is what the roofline needs
    calls = 0
    stage_ms = [0.0, 0.0, 0.0]
    if not args.no_stage_profile:
        _, _, stage_ms, calls, _ = timed(profile=True, per_step=False)
    # per-step distribution (events around every step: no PDL overlap across steps)
    _, step_ms, _, _, _ = timed(profile=False, per_step=True)
    graph_ms = timed_graph() if args.graph and args.l2 == "rotate" else None
    # secondary: warm L2 -- the same copy every step, when the step's
    # Enc(W) fits in half the L2; rank-local, no barrier
    warm_ms = None
    if enc_bytes * 2 <= l2_bytes and ws_batch is None:
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        for _ in range(args.steps):
            step()
        b_.record(stream)
        torch.cuda.synchronize()
        warm_ms = a_.elapsed_time(b_) / args.steps

    # ---------------- e2e through the host-buffer C-ABI call (H2D X + D2H cts,R inside)
    e2e = None
    if not args.no_e2e:
        hosts = []
        # consecutive matmuls with one input that the library runs as one resident-X group (Q, K, V
        # at k <= 128, ell <= 16, m <= 768, R > 1) get ONE pinned copy, uploaded once per group;
        # every other matmul gets its own copy (and its own upload)
        pinned = []
        prev = None
        for mt in mats:
            lay = mt["lay"]
            grp = cfg.ell <= 16 and lay.k <= 128 and lay.m <= 768 and 2 * lay.n <= cfg.N
            key = mt["X"][0].data_ptr()
            if grp and prev is not None and prev[0] == key:
                Xh = prev[1]
            else:
                Xh = mt["X"][0].cpu().pin_memory()
                pinned.append(Xh)
            prev = (key, Xh) if grp else None
            if wide:
                c_, R_ = nb.alloc_outputs_u64(ctx, mt["encw"][0], lay.k_per_query, lay.n_queries)
                ch, Rh = c_.cpu().pin_memory(), R_.cpu().pin_memory()
            else:
                ch, Rh = nb.alloc_outputs(ctx, mt["encw"][0], lay.k_per_query, lay.n_queries, pin=True,
                                          device="cpu")
            hosts.append((Xh, ch, Rh))
        h2d = sum(x.numel() * x.element_size() for x in pinned)
        d2h = sum(h[1].numel() * h[1].element_size() + h[2].numel() * h[2].element_size() for h in hosts)
        host_matmul = nb.nimbus_cop_matmul_host_u64 if wide else nb.nimbus_cop_matmul_host

        # (1) headline: K steps through the pipelined host-buffer call, one call for the whole
        # sequence (every step uploads its X and downloads its ciphertexts and R; the copies of
        # step i+1 / i-1 overlap the compute of step i); Enc(W) copies rotate as in pass A
        def host_jobs(nsteps, first):
            jobs = []
            for i in range(nsteps):
                c = (first + i) % n_copies
                for mt, (Xh, ch, Rh) in zip(mats, hosts):
                    lay = mt["lay"]
                    jobs.append(dict(encw=mt["encw"][c], X=Xh, k_per_query=lay.k_per_query,
                                     n_queries=lay.n_queries, mask_seed=mt["seed"], cts=ch, R=Rh))
            return jobs
        ke = max(3, min(args.steps, 50))
        jobs_t = host_jobs(ke, 0)
        ws_h = torch.empty(nb.nimbus_cop_workspace_size_host_batch(ctx, jobs_t, wide=wide), dtype=torch.uint8,
                           device=dev)
        nb.nimbus_cop_matmul_host_batch(ctx, host_jobs(max(3, min(args.warmup, 10)), 1), ws_h, wide=wide)
        e2e_runs = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nb.nimbus_cop_matmul_host_batch(ctx, jobs_t, ws_h, wide=wide)   # synchronises before returning
            e2e_runs.append((time.perf_counter() - t0) * 1e3 / ke)
        e2e_step = max_over_ranks(statistics.median(e2e_runs), world, dev)
        del ws_h

        # (2) latency of ONE synchronous host-buffer call per step (cold L2 before each)
        def step_host():
            c = step_no[0] % n_copies
            for mt, (Xh, ch, Rh) in zip(mats, hosts):
                lay = mt["lay"]
                host_matmul(ctx, mt["encw"][c], Xh, lay.k_per_query, lay.n_queries, mt["seed"],
                            ch, Rh, mt["ws"])
        for _ in range(3):
            cold()
            step_host()
        single_ms = []
        for _ in range(max(3, min(args.steps, 20))):
            cold()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step_host()                      # synchronises the stream before returning
            single_ms.append((time.perf_counter() - t0) * 1e3)
        single_step = max_over_ranks(statistics.median(single_ms), world, dev)
        e2e = dict(step_ms=e2e_step, h2d=h2d, d2h=d2h, single_ms=single_step, steps=ke)
    l2_desc = (f"cold: {n_copies} rotating copies of Enc(W)+X ({n_copies * enc_bytes >> 20} MiB >= 3x the "
               f"{l2_bytes >> 20} MiB L2), step i reads copy i mod {n_copies}" if args.l2 == "rotate" else
               f"flushed by a {L2_FLUSH_BYTES >> 20} MiB write before every timed step")
    if args.prefetch_next and cfg.ell <= 16 and max(l.k for _, _, l in cfg.layers) <= 128:
        l2_desc += ("; nimbus_cop_prefetch_next names the next step's Enc(W) copy: each contraction CTA prefetches the next "
                    "launch's first two tiles (28 of 50 MB) into L2 after its own last copy is issued (--prefetch-next 0: off)")
    return dict(total_ms=total_ms, step_ms=step_ms, stage_ms=stage_ms, calls=calls, launches=launches, graph_ms=graph_ms,
                kernel=kernel,
                clocks=clk, t_setup=t_setup, enc_bytes=enc_bytes, e2e=e2e, l2_desc=l2_desc, warm_ms=warm_ms,
                setup=dict(gpu_ms=setup_gpu_ms, host_s=setup_host_s, bytes=setup_bytes))


# ----------------------------------------------------------------- CPU oracle
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg, budget_s, rows_cap=None):
    """Time the oracle (as it stands) on a bounded row sample of the workload:
    the first matrix of the config, steps 2-4 on `rows` rows (whole packed
    groups), grown until ~budget_s of CPU work.  Returns (modMAC/s, desc)."""
    from oracle import oracle as O
    li, pj, lay = cfg.layers[0]
    seed = ni.seed_mm(cfg.cid, li, pj)
    pr = O.primes(cfg.N, cfg.L)
    s = O.keygen(cfg.N, cfg.seed_cfg)
    W = ni.gen_W(seed, lay.m, lay.n, cfg.ell)
    t0 = time.perf_counter()
    E = O.encrypt_rows(cfg.N, cfg.L, pr, cfg.ell, s, W, seed)
    t_enc = time.perf_counter() - t0
    R = cfg.N // lay.n
    rows = min(lay.k_per_query, R)
    done_macs, done_t, reps = 0, 0.0, 0
    while True:
        X = ni.gen_X(seed, rows, lay.m, cfg.ell)
        t0 = time.perf_counter()
        O.cop_matmul(cfg.N, cfg.L, cfg.L_out, pr, cfg.ell, E, X, lay.n, rows, 1, seed)
        dt = time.perf_counter() - t0
        done_macs += ni.modmacs(rows, lay.m, cfg.N, cfg.L)
        done_t += dt
        reps += 1
        if done_t >= budget_s or (rows_cap and rows >= rows_cap):
            break
        if rows < lay.k_per_query:
            rows = min(lay.k_per_query, rows * 2)
    desc = (f"{cfg.name} matrix {lay.name} (m={lay.m}, n={lay.n}): oracle steps 2-4 on up to {rows} rows "
            f"x {reps} runs, {done_t:.1f} s CPU wall; Enc(W) setup {t_enc:.1f} s untimed")
    return done_macs / done_t, desc


def cpu_baseline(cfg, budget_s):
    """The oracle as it stands, on the host's cores (all of them, then one thread;
    BASELINE.md §3): a reported baseline, not the target."""
    if cfg.ell > 32:
        # q > 2^128: only the Python-integer oracle (oracle/wide.py) covers ell = 64, far too slow
        # to time on a workload-sized sample
        return {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "cpu_model": cpu_model(),
                "sample": "not timed: the ell > 32 oracle is Python integers (oracle/wide.py)"}
    from oracle import oracle as O
    all_threads = O.set_threads(os.cpu_count() or 1)
    v, desc = oracle_sample(cfg, budget_s)
    O.set_threads(1)
    v1, desc1 = oracle_sample(cfg, budget_s / 2)
    O.set_threads(all_threads)
    return {"value": v, "unit": UNIT, "cores": all_threads, "kind": "oracle", "sample": desc,
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": desc1}}


def workload_config(cfg):
    """The workload keys both arms print identically (the driver compares them)."""
    lays = [l for _, _, l in cfg.layers]
    return {"workload": workload_name(cfg), "config": cfg.name, "k": lays[0].k, "matmuls_per_step": len(lays)}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return None
    if cfg.ell > 32:
        return {"impl": "reference", "unavailable": "ell > 32 needs the Python-integer oracle (oracle/wide.py), "
                                                    "not timed as a reference arm"}
    from oracle import oracle as O
    cores = O.set_threads(os.cpu_count() or 1)
    li, pj, lay = cfg.layers[0]
    seed = ni.seed_mm(cfg.cid, li, pj)
    pr = O.primes(cfg.N, cfg.L)
    s = O.keygen(cfg.N, cfg.seed_cfg)
    W = ni.gen_W(seed, lay.m, lay.n, cfg.ell)
    E = O.encrypt_rows(cfg.N, cfg.L, pr, cfg.ell, s, W, seed)
    R = cfg.N // lay.n
    # calibrate one packed group, then size each step so the run stays ~ within 120 s
    rows = min(R, lay.k_per_query)
    X = ni.gen_X(seed, rows, lay.m, cfg.ell)
    t0 = time.perf_counter()
    O.cop_matmul(cfg.N, cfg.L, cfg.L_out, pr, cfg.ell, E, X, lay.n, rows, 1, seed)
    t1 = time.perf_counter() - t0
    per_row = t1 / rows
    budget = 120.0 / max(1, args.steps + args.warmup)
    rows = int(max(1, min(lay.k_per_query, budget / per_row)))
    X = ni.gen_X(seed, rows, lay.m, cfg.ell)
    for _ in range(args.warmup):
        O.cop_matmul(cfg.N, cfg.L, cfg.L_out, pr, cfg.ell, E, X, lay.n, rows, 1, seed)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.cop_matmul(cfg.N, cfg.L, cfg.L_out, pr, cfg.ell, E, X, lay.n, rows, 1, seed)
        times.append(time.perf_counter() - t0)
    macs = ni.modmacs(rows, lay.m, cfg.N, cfg.L)
    value = macs * len(times) / sum(times)
    sample = (f"{rows} of {lay.k} rows of {cfg.name} matrix {lay.name} per step (oracle steps 2-4: "
              f"contraction + packing + mod-switch + mask), {cores} OpenMP threads")
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u128", "data": "synthetic",
            "config": workload_config(cfg),
            "impl": "reference", "impl_detail": "reference (oracle/, CPU)", "sample_rows": rows,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------- roofline
def algorithmic_bytes(cfg, lay):
    """SURVEY.md §8(d) bytes of one matmul: Enc(W) + X in + compact output ciphertexts + R out."""
    es = 4 if cfg.ell <= 32 else 8
    nct = lay.n_queries * -(-lay.k_per_query // (cfg.N // lay.n))
    return (lay.m * 2 * cfg.L * cfg.N * 4 + lay.k * lay.m * es + nct * 2 * cfg.L_out * cfg.N * 4
            + lay.k * lay.n * es)


def i8_floor():
    """The measured tcgen05 kind::i8 rate (tools/mma_bench.cu, profiles/mma_bench.json), if captured."""
    path = os.path.join(ROOT, "profiles", "mma_bench.json")
    if os.path.exists(path):
        d = json.load(open(path))
        if d.get("tops_n256"):
            return float(d["tops_n256"]), d.get("src", "profiles/mma_bench.json")
    return None, None


def ncu_traffic(cfg, kernel):
    """DRAM read+write bytes per launch from profiles/ncu_<config>.json, when its captured kernel
    is the kernel this line ran."""
    path = os.path.join(ROOT, "profiles", f"ncu_{cfg.name.replace('@', '')}.json")
    if not os.path.exists(path):
        return None, None
    cap = json.load(open(path)).get("kernel_capture", {})
    name = (cap.get("kernel") or "").replace("void ", "").split("(")[0].replace("(int)", "").replace(" ", "")
    if name.startswith("k_cop_pk<"):      # the library prints the CTA-pair flag (4th parameter) as "", ", P2"
        name = name[:-3] + ">" if name.endswith(",0>") else name[:-3] + ",P2>" if name.endswith(",1>") else name
    if cap.get("dram_traffic_bytes") is None or name != kernel.replace(" ", ""):
        return None, f"profiles/ncu_{cfg.name}.json captured {name or '?'}, not {kernel}"
    return cap["dram_traffic_bytes"], f"profiles/ncu_{cfg.name.replace('@', '')}.json ({name})"


def make_line(args, cfg, res, world, steps, warmup, cpu):
    """The JSON record of one config: the contract keys plus roofline, e2e, cpu_baseline."""
    peaks = measured_peaks()
    lays = [l for _, _, l in cfg.layers]
    macs_step = sum(ni.modmacs(l.k, l.m, cfg.N, cfg.L) for l in lays)
    ms_step = res["total_ms"] / steps
    value = weak_value(macs_step, world, ms_step)
    # roofline of the dominant kernel (the contraction, stage 1), per launch: the per-step units
    # (modMACs -> int8 ops, §8(d) bytes) over the contraction launches of a step
    SX, SW = sx_of(cfg.ell), 4
    launches_step = max(1.0, res["calls"] / steps) if res["calls"] else float(len(lays))
    contract_ms = res["stage_ms"][1] / res["calls"] if res["calls"] else 0.0
    if contract_ms <= 0:   # stage events off: bound the kernel by the whole step (conservative)
        contract_ms = ms_step / launches_step
    ops = 2 * macs_step * SX * SW / launches_step                          # int8 tensor ops per launch
    hbm_bytes = sum(algorithmic_bytes(cfg, l) for l in lays) / launches_step
    long_step = ms_step > 5.0   # a kernel timed inside a long (multi-matmul) step: sustained peak
    i8_peak = 2.0 * (peaks["bf16_tflops_sustained"] if long_step else peaks["bf16_tflops"])
    floor, fsrc = i8_floor()
    # which ceiling binds: the tensor time at the kernel's real int8 rate (the measured kind::i8
    # floor when captured, else the 2 x bf16 figure) against the HBM time of the §8(d) bytes
    t_i8 = ops / ((floor or i8_peak) * 1e12)
    t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9)
    tens = {"bound": "tensor", "achieved": ops / (contract_ms / 1e3) / 1e12, "peak": i8_peak, "unit": "TFLOP/s"}
    tens["frac"] = tens["achieved"] / tens["peak"]
    hbm = {"bound": "hbm", "achieved": hbm_bytes / (contract_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
           "unit": "GB/s"}
    hbm["frac"] = hbm["achieved"] / hbm["peak"]
    prim, alt = (tens, hbm) if t_i8 >= t_hbm else (hbm, tens)
    prim = dict(prim)
    kernel = res.get("kernel") or "?"
    prim["traffic"], src = (ncu_traffic(cfg, kernel) if args.impl == "tcgen05" else (None, None))
    if src:
        prim["traffic_src"] = src
    # DRAM bytes per step of the chained pass itself (ncu range replay over K block-timed steps,
    # profiles/range_traffic.json): what the steps move when they run as timed, PDL-overlapped and
    # with the L2 as the previous step left it -- a --set full capture replays one serialised launch
    rt_path = os.path.join(ROOT, "profiles", "range_traffic.json")
    if args.impl == "tcgen05" and os.path.exists(rt_path):
        ent = json.load(open(rt_path)).get(cfg.name, {}).get(f"prefetch_next={args.prefetch_next}")
        if ent:
            prim["traffic_chain"] = ent["dram_bytes_per_step"] / launches_step
            prim["traffic_chain_src"] = "profiles/range_traffic.json (ncu --replay-mode range over the block-timed steps)"
    prim["kernel"] = kernel
    prim["launch_ms"] = contract_ms
    prim["launches_per_step"] = launches_step
    prim["peak_src"] = (f"{peaks['src']}: int8 = 2 x bf16 {'sustained' if long_step else 'burst'} (guide's nominal ratio)"
                        if prim["bound"] == "tensor" else f"{peaks['src']} hbm_gbs")
    prim["units_per_launch"] = ({"int8_ops": ops} if prim["bound"] == "tensor" else
                                {"bytes": hbm_bytes, "bytes_def": "|Enc(W)| + |X| + |compact cts| + |R| (SURVEY.md §8(d))"})
    step_units = (ops if prim["bound"] == "tensor" else hbm_bytes) * launches_step
    step_ach = step_units / (ms_step / 1e3) / (1e12 if prim["bound"] == "tensor" else 1e9)
    step_roof = {"bound": prim["bound"], "achieved": step_ach, "peak": prim["peak"], "unit": prim["unit"],
                 "frac": step_ach / prim["peak"], "ms": ms_step}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(cfg),
        "impl": args.impl, "l2": res["l2_desc"], "enc_w_bytes_resident": res["enc_bytes"],
        "roofline": prim,
        "roofline_other": alt,
        # the whole step against the same ceiling: the step's units over ms_per_step of the timed pass
        # (all kernels of the step, PDL-chained, no event between them), not one bracketed launch
        "roofline_step": step_roof,
        "roofline_i8_floor": (None if floor is None else
                              {"achieved": tens["achieved"], "peak": floor, "unit": "TFLOP/s",
                               "frac": tens["achieved"] / floor, "peak_src": fsrc}),
        "stages_ms_per_step_profiled": {"slice_x": res["stage_ms"][0] / steps,
                                        "contraction": res["stage_ms"][1] / steps,
                                        "pack_moddown_mask": res["stage_ms"][2] / steps},
        # per-step spread of the timed pass (CUDA events around each step, rank 0)
        "step_ms_dist": dict(step_dist(res["step_ms"]),
                             note="separate pass, CUDA events around every step (no PDL overlap across steps)"),
        # secondary: Enc(W) L2-resident (same copy every step); null when it does not fit
        "warm_l2": (None if res["warm_ms"] is None else
                    {"ms_per_step": res["warm_ms"], "value": weak_value(macs_step, 1, res["warm_ms"]),
                     "unit": UNIT}),
        "graph": (None if res["graph_ms"] is None else
                  {"ms_per_step": res["graph_ms"], "value": weak_value(macs_step, world, res["graph_ms"]),
                   "unit": UNIT, "note": "secondary: the same steps replayed from a CUDA graph capturing n_copies "
                           "consecutive steps (one per input copy)"}),
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "setup_encrypt_s": res["t_setup"],
        # Alg. 1 step 1 for the first matrix, steady state: Enc(W) bytes written / GPU time
        "setup": {"matrix": f"{lays[0].m}x{lays[0].n}", "enc_w_bytes": res["setup"]["bytes"],
                  "gpu_ms": res["setup"]["gpu_ms"], "host_ms": res["setup"]["host_s"] * 1e3,
                  "gb_per_s": res["setup"]["bytes"] / (res["setup"]["gpu_ms"] * 1e-3) / 1e9,
                  "hbm_frac": res["setup"]["bytes"] / (res["setup"]["gpu_ms"] * 1e-3) / 1e9 / peaks["hbm_gbs"]},
    }
    if res["e2e"] is not None:
        e = res["e2e"]
        out["e2e"] = {"value": weak_value(macs_step, world, e["step_ms"]), "unit": UNIT,
                      "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"], "ms_per_step": e["step_ms"],
                      "call": f"nimbus_cop_matmul_host_batch: {e['steps']} steps in one pipelined call (pinned host "
                              f"X in, ciphertexts + R out every step; Enc(W) copies rotate), wall clock / steps",
                      "single_call": {"ms_per_step": e["single_ms"],
                                      "value": weak_value(macs_step, world, e["single_ms"]),
                                      "call": "one synchronous nimbus_cop_matmul_host per matmul, L2 cold before"}}
    if cpu:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_budget_s)
    return out


def bench_config(args, key, rank, world, local_rank, steps=None, warmup=None, e2e=True, cpu=True):
    """Run and describe one config; frees its device memory before returning."""
    import copy
    import gc
    import torch
    cfg = get_config(key)
    a = copy.copy(args)
    a.steps = args.steps if steps is None else steps
    a.warmup = args.warmup if warmup is None else warmup
    a.no_e2e = args.no_e2e or not e2e
    res = run_gpu(a, cfg, rank, world, local_rank)
    gc.collect()
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    return make_line(a, cfg, res, world, a.steps, a.warmup, cpu and world == 1 and not args.no_cpu_baseline)


# ----------------------------------------------------------------- main
MAIN_CONFIG = "5"
# (config, steps cap, steps floor) of the per_config block: the single-matmul configs (20 us .. 0.6 ms per
# step) at >= 200 steps -- 20 steps are a few ms, inside one swing of the power-capped clock right after
# the C5 pass (C4 ran 198-238 us per step that way, 4 runs) -- the C5@l16 pass and the paper's ell = 64
# pass at <= 5 steps (a 27 GB Enc(W), ~0.3 s per pass).  Each entry states its own steps / warmup.
PER_CONFIG = (("2", None, 200), ("2qkv", None, 200), ("3", None, 200), ("4", None, 200), ("4l16", None, 200),
              ("5l16", 5, 0), ("4l64", None, 200), ("5l64", 5, 0))


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    key = args.config or MAIN_CONFIG
    cfg = get_config(key)
    if args.impl == "reference":
        out = run_reference(args, cfg, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    line = bench_config(args, key, rank, world, local_rank)
    if args.config is None and args.per_config:
        per = {}
        for k2, cap, floor in PER_CONFIG:
            st = max(args.steps, floor) if cap is None else min(args.steps, cap)
            wu = args.warmup if cap is None else min(args.warmup, 3)
            d = bench_config(args, k2, rank, world, local_rank, steps=st, warmup=wu)
            if d is not None:
                per[get_config(k2).name] = d
        if line is not None:
            line["per_config"] = per
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
