#!/usr/bin/env python
"""Benchmark: one QEM iteration (sample -> MPIW E-step -> EMA/M-step) per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

  --gpus N > 1 without a torchrun environment re-launches itself under
  `python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL).

Contract:
  * a step is one whole hot-path pass = one QEM iteration (Alg. 1):
    Philox sampler (K1; fused into the column prep on the tensor-core path) -> forward pair
    tiles (K2) -> [NCCL all-reduce of the
    (K+1) fp64 plate sums when N > 1, run inside libqem: qem_estep_reduce] -> root +
    backward weights/moments (K3, K4)
    -> EMA + M-step (K5), on BASELINE config C (default 5; config 4 with --config 4);
  * metric: E-step factor-pairs/s (N*K^2 per step over the whole iteration), plus
    QEM iterations/s; strong scaling (the config's M groups split over N ranks);
  * timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
    CUDA events on the launching stream, max over ranks; inputs exceed L2;
  * roofline: the dominant kernel's pair rate vs the ALU ceiling;
  * e2e: the same iteration through the public API with the observations
    copied host->device from pinned memory and log Pe + Q read back every step;
  * cpu_baseline: the fp64 CPU oracle on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic per-pair counts: per pass, d+2 FP32 ops + 1 exp.
SFU_PER_SM_CLK = 16.0     # MUFU.EX2 lanes/clk/SM (guide; measured 15.3, profiles/r01_microbench_pipes.txt)
FP32_PER_SM_CLK = 128.0   # FFMA lanes/clk/SM (guide; measured 124-126)
SMS = 148
SM_MAX_MHZ = 1965.0


# FMA-pipe lane-ops of one exponential evaluated in software (exp2_poly2: 3 FADD + 5 FFMA;
# the 2 integer ops of the exponent insert run on the ALU pipe)
FMA_PER_SOFT_EXP = 8.0


def exp_capacity(fma_other: float, mhz: float = SM_MAX_MHZ) -> dict:
    """Pairs/s ceiling of ONE pass when every pair needs one exponential plus `fma_other` FMA-pipe
    lane-ops, and the exponentials may run on the SFU (16 MUFU.EX2/clk/SM) or in software on the
    FMA pipe (128 lane-ops/clk/SM, FMA_PER_SOFT_EXP each): maximise P subject to
    (1 - f) P <= 16 and P (fma_other + 8 f) <= 128 over the software fraction f."""
    f = max(0.0, (FP32_PER_SM_CLK - SFU_PER_SM_CLK * fma_other) / (SFU_PER_SM_CLK * FMA_PER_SOFT_EXP + FP32_PER_SM_CLK))
    p = min(SFU_PER_SM_CLK / (1.0 - f), FP32_PER_SM_CLK / (fma_other + FMA_PER_SOFT_EXP * f))
    return {"pairs_per_clk_sm": p, "soft_exp_fraction": f, "pairs_per_s": p * mhz * 1e6 * SMS}


def pair_ceiling(d: int, tc: bool = False, mhz: float = SM_MAX_MHZ) -> dict:
    """Pairs/s ceiling of ONE pass (forward or backward) from the binding resources.

    FFMA tiles (tc False): 1 exp + d+2 FP32 lane-ops per pair.
    tcgen05 tiles (tc True, d = 16): the d-term contraction runs on the tensor cores (bf16x3:
    6 bf16 products = 12 d flops/pair, ceiling from the measured bf16 peak), leaving 1 exp + 2
    FMA-pipe lane-ops per pair for the SM (the forward: subtract the running max, accumulate; the
    backward folds its column constant into the MMA and needs only the accumulate, so this is
    the forward's -- the dominant kernel's -- ceiling).
    Binding ceiling = the exp capacity of SFU + FMA pipe together (exp_capacity); the SFU-only
    figure (16 pairs/clk/SM) is reported beside it."""
    f = mhz * 1e6 * SMS
    other = 2.0 if tc else d + 2.0
    cap = exp_capacity(other, mhz)
    # north-star roofline (BASELINE.json): the slower of the SFU ops (1 exp per pair) and the FP32
    # ops (`other` per pair) at peak; HBM is < 5 % of any pair kernel (DESIGN.md Roofline)
    sfu, fp32 = f * SFU_PER_SM_CLK, f * FP32_PER_SM_CLK / other
    out = {"sfu_pairs_per_s": sfu, "fp32_pairs_per_s": fp32,
           "exp_sfu_plus_fma_pairs_per_s": cap["pairs_per_s"], "soft_exp_fraction_at_ceiling": cap["soft_exp_fraction"]}
    pipes = {"sfu": sfu, "fp32": fp32}
    if tc:
        out["tensor_pairs_per_s"] = pipes["tensor"] = BF16_TFLOPS * 1e12 / (12.0 * d)
    pipe = min(pipes, key=pipes.get)
    out.update(pairs_per_s=pipes[pipe], pipe=pipe)
    return out


def _measured_bf16() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0  # nominal dense bf16 (B200_PROFILING.md fallback)


BF16_TFLOPS = _measured_bf16()


def _ncu_traffic(kernel: str, cfg: int):
    """DRAM bytes per launch of `kernel` on config `cfg` from the committed ncu --set full capture
    (tools/ncu_traffic.py -> profiles/r02_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            return json.load(f)[f"config{cfg}"][kernel]["dram_bytes"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=1)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- CPU oracle


def oracle_sample(cfg: int, budget_s: float = 15.0, threads: int | None = None):
    """Time the fp64 oracle E-step + EMA (as it stands) on a bounded sample of groups of config ``cfg``
    with `threads` OpenMP threads (default: all host cores).

    Returns (pairs/s, iters/s extrapolated to the full config, threads, description)."""
    from oracle import oracle as orc
    from paper_2503_08264_b200 import synth
    full = synth.config(cfg)
    cores = threads or os.cpu_count() or 1
    orc.set_num_threads(cores)
    n = max(1, min(full.n, cores))
    spent, done_pairs, n_runs = 0.0, 0, 0
    while True:
        m = synth.config(cfg, n=n)
        data = synth.make_data(m)
        q = synth.initial_q(m)
        eps = orc.eps_for_iteration(m, 1, 100 + cfg)
        state = orc.initial_state(m)
        t0 = time.perf_counter()
        orc.qem_step(m, state, q, eps, 1, data=data)
        dt = time.perf_counter() - t0
        spent += dt
        done_pairs += m.pairs
        n_runs += 1
        if spent > budget_s * 0.3 or n >= full.n:
            break
        # grow the sample towards the budget
        n = min(full.n, max(n + 1, int(n * min(8.0, (budget_s * 0.3) / max(dt, 1e-3)))))
    pairs_per_s = done_pairs / spent
    iters_per_s = pairs_per_s / full.pairs
    desc = (f"oracle fp64 E-step+EMA of config {cfg} on {n} of {full.n} groups (K={full.K}), "
            f"{n_runs} run(s), {spent:.1f} s, OpenMP threads={orc.num_threads()}; iters/s extrapolated "
            f"to all {full.n} groups")
    return pairs_per_s, iters_per_s, orc.num_threads(), desc


# ---------------------------------------------------------------- GPU bench


def _algo_bytes_method(dom: str, n: int, m) -> float:
    """The METHOD's bytes for one launch of the dominant pair kernel (SURVEY.md §8(d) "Bytes per
    E-step": samples read, the unary term, messages / weights written), independent of how the
    kernel lays out its operands: per (group, sample) the d fp32 sample coordinates + the fp32
    unary log-term (P or ln P) in, and the pass's output out (forward: the message g; backward:
    the weight w), 4 B each."""
    return float(n) * m.K * (4.0 * m.d + 4.0 + 4.0)


def measure_step(m, args, world, rank, dev, in_library, seed):
    """Device-timed QEM iterations of model `m` (groups sharded over `world` ranks): W warm-up
    steps, then K steps bracketed by barrier + synchronize; CUDA events on the launch stream;
    per-kernel events around the two pair kernels (recorded by libqem); max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.dist import ShardedQEM
    from paper_2503_08264_b200.qem import QEM, shard_range

    data = synth.make_data(m)
    gb, ge = shard_range(m.n, rank, world)
    g = QEM(m, group_begin=gb, group_end=ge, device=dev)
    g.set_data(data)
    stream = torch.cuda.current_stream()
    runner = ShardedQEM(g, in_library=in_library)
    launched = [0]

    def step(t, ev=None):
        # ev: [fwd kernel start, fwd kernel end, bwd kernel start, bwd kernel end, allreduce start, end]
        if ev:
            g.set_kernel_events(ev[:4])
        g.sample_estep_forward(seed, t)  # sampler + forward (the draws fused into the column prep on the TC path)
        launched[0] += g.kernel_launches()
        if ev:
            ev[4].record(stream)
        runner.allreduce_plate_sum()
        if ev:
            ev[5].record(stream)
        g.estep_backward()
        launched[0] += g.kernel_launches()
        g.mstep(t)
        launched[0] += g.kernel_launches()

    t = 1
    for _ in range(args.warmup):
        step(t)
        t += 1
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    local = dev.index or 0
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launched[0] = 0
    g.mode_hist()  # read-and-reset: the timed steps' forward tile modes only
    start.record(stream)
    for s in range(args.steps):
        step(t, evs[s])
        t += 1
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    hist = g.mode_hist()
    ms_total = start.elapsed_time(stop)
    g.set_kernel_events(None)
    fwd_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    bwd_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    comm_ms = sum(e[4].elapsed_time(e[5]) for e in evs) / args.steps
    flags, clamps = g.read_flags()
    if world > 1:
        tt = torch.tensor([ms_total, fwd_ms, bwd_ms, comm_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total, fwd_ms, bwd_ms, comm_ms = tt.tolist()
    ms_step = ms_total / args.steps
    tc = g.pair_path() == 1
    local_pairs = (ge - gb) * m.K * m.K
    dom, dom_ms = ("forward", fwd_ms) if fwd_ms >= bwd_ms else ("backward", bwd_ms)
    kname = f"k_{dom}" + ("_tc" if tc else "")
    ceil = pair_ceiling(m.d, tc)
    achieved = local_pairs / (dom_ms * 1e-3)
    per_pair = ({"exp": 1, "fma_pipe": 2, "tensor_bf16_flops": 12 * m.d} if tc else {"exp": 1, "fma_pipe": m.d + 2})
    algo = _algo_bytes_method(dom, ge - gb, m)
    traffic = _ncu_traffic(kname, args.config if m.config_id == args.config else m.config_id)
    roof = {"bound": "alu", "pipe": ceil["pipe"], "kernel": kname, "unit": "Gpair/s",
            "achieved": achieved / 1e9, "peak": ceil["pairs_per_s"] / 1e9,
            "frac": achieved / ceil["pairs_per_s"],
            "frac_vs_exp_sfu_plus_fma": achieved / ceil["exp_sfu_plus_fma_pairs_per_s"],
            "traffic": traffic,
            "traffic_unit": "DRAM bytes/launch (ncu --set full, profiles/r02_traffic.json)",
            "algorithmic_bytes": algo,
            "algorithmic_bytes_basis": "SURVEY.md §8(d): per (group, sample) d fp32 coordinates + the fp32 unary "
                                       "term in, the pass's fp32 output out",
            "traffic_over_algorithmic": (traffic / algo) if traffic else None,
            "achieved_gbs_algorithmic": algo / (dom_ms * 1e-3) / 1e9,
            "per_pair": per_pair,
            "ceilings_gpair_s": {k.replace("_pairs_per_s", ""): v / 1e9 for k, v in ceil.items()
                                 if k.endswith("_pairs_per_s") and k != "pairs_per_s"},
            "peak_basis": (f"{SMS} SMs x {SM_MAX_MHZ:.0f} MHz x min({SFU_PER_SM_CLK:.0f} MUFU.EX2/clk per exp, "
                           f"{FP32_PER_SM_CLK:.0f} FP32 lane-ops/clk / {per_pair['fma_pipe']} per pair) = the north-star "
                           f"roofline (slower of SFU and FP32 ops at peak, guide peak rates); "
                           f"frac_vs_exp_sfu_plus_fma is against the stricter ceiling that also counts exps "
                           f"evaluated in software on the FMA pipe ({FMA_PER_SOFT_EXP:.0f} lane-ops each)"),
            "kernels_ms": {"forward": fwd_ms, "backward": bwd_ms, "allreduce": comm_ms},
            "forward_mode_hist": dict(zip(["expm1_deg3", "deg4", "deg5", "deg7", "deg9", "online_lse"],
                                          [int(x) for x in hist[:6]])),
            "backward_moment_groups": int(hist[6]),
            "forward_lazy_max_redos": int(hist[7])}
    out = dict(g=g, data=data, gb=gb, ge=ge, ms_step=ms_step, value=m.pairs / (ms_step * 1e-3),
               launched=launched[0], flags=flags, clamps=clamps, clocks=clk, roofline=roof, tc=tc, t=t,
               allreduce=runner.allreduce_plate_sum, nccl=g.nccl_info() if in_library else None)
    return out


def _summary(meas, m):
    """The JSON-able part of a measure_step result."""
    return {"workload": f"config{m.config_id}:{m.name}", "M_groups": m.n, "K": m.K, "d": m.d, "J": m.J,
            "pairs_per_step": m.pairs, "ms_per_step": meas["ms_step"], "value": meas["value"],
            "unit": "factor-pairs/s", "qem_iters_per_s": 1e3 / meas["ms_step"], "roofline": meas["roofline"],
            "gpu_launches": meas["launched"], "flags": {"device_flags": meas["flags"], "var_clamps": meas["clamps"]},
            "clocks": meas["clocks"]}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2503_08264_b200 import synth

    world, rank, local = dist_env()
    if world > 1 and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m = synth.config(args.config)
    seed = 100 + args.config
    main_m = measure_step(m, args, world, rank, dev, in_library=world > 1, seed=seed)
    g = main_m["g"]

    # ------------------------------------------------------------- e2e leg
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, g, m, main_m["data"], world, rank, dev, seed, main_m["t"], main_m["allreduce"])
    nccl = main_m["nccl"]
    g.close()
    variants = {}
    if not args.no_variants:
        # config 4 (the other gated config) at the same world size, sharded the same way
        other = 4 if args.config == 5 else (5 if args.config == 4 else None)
        if other is not None:
            mo = synth.config(other)
            meas = measure_step(mo, args, world, rank, dev, in_library=world > 1, seed=100 + other)
            meas["g"].close()
            variants[f"config{other}"] = _summary(meas, mo)
        if world == 1:
            variants["converged_regime"] = run_converged_variant(args, dev)
            variants["iterate_graph"] = run_iterate_variant(dev)
            variants["fresh_denominator"] = run_fresh_variant(args, m, main_m["data"], dev, seed)
            variants["mstep_family"] = run_mstep_family_variant(dev)
            variants["discrete_occupancy"] = run_discrete_variant(dev)
            variants["predictive_loglik"] = run_predictive_variant(m, main_m["data"], dev, seed)
            variants["gamma_poisson"] = run_gamma_variant(dev)
            variants["crossed_bus"] = run_crossed_variant(dev)
            variants["qmp_nonfactorised"] = run_qmp_variant(dev)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, args.cpu_budget)
    ms_step = main_m["ms_step"]
    line = {
        "metric": "E-step factor-pairs/sec (N*K^2) and QEM iters/sec",
        "value": main_m["value"],
        "unit": "factor-pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": DTYPE_TC if main_m["tc"] else DTYPE_FFMA,
        "data": "synthetic (ancestral draw from the config's prior, numpy PCG64 seed = config id)",
        "qem_iters_per_s": 1e3 / ms_step,
        "config": {"workload": f"config{args.config}:{m.name}", "M_groups": m.n, "K": m.K, "d": m.d,
                   "J": m.J, "pairs_per_step": m.pairs, "parallelism": f"groups sharded over {world} rank(s)",
                   "allreduce": ("in-library ncclAllReduce of K+1 fp64 (qem_estep_reduce)" if world > 1 else "none (1 rank)"),
                   "nccl": ({"rank": nccl[0], "nranks": nccl[1], "version": nccl[2]} if nccl else None),
                   "l2": "inputs larger than L2 (samples + per-group messages > 126 MB)",
                   "sampler": "device Philox4x32-10",
                   "regime": "early run from Q = N(0,1): timed from iteration W+1 (converged regime in variants)"},
        "roofline": main_m["roofline"],
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": main_m["launched"],
        "clocks": main_m["clocks"],
        "flags": {"device_flags": main_m["flags"], "var_clamps": main_m["clamps"]},
        "variants": variants,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


DTYPE_TC = ("f32 (config-5 log-factor contraction: bf16x3 split on tcgen05, fp32 TMEM accumulation; "
            "exp fp32: SFU ex2.approx + 2/16 fwd, 4/16 bwd degree-5 polynomial; f64 unary terms, plate sums, moments)")
DTYPE_FFMA = "f32 pair tiles (FFMA + SFU ex2.approx), f64 unary terms, plate sums, moments"


def cpu_baseline(cfg, budget):
    """The fp64 oracle as it stands, on a bounded sample of the workload, at all host cores and at 1 thread."""
    try:
        cores = os.cpu_count() or 1
        pps, ips, used, desc = oracle_sample(cfg, budget_s=budget, threads=cores)
        out = {"value": pps, "unit": "factor-pairs/s", "cores": used, "kind": "oracle", "sample": desc,
               "qem_iters_per_s": ips}
        p1, i1, _, d1 = oracle_sample(cfg, budget_s=max(4.0, budget / 3), threads=1)
        out["one_thread"] = {"value": p1, "unit": "factor-pairs/s", "cores": 1, "sample": d1, "qem_iters_per_s": i1}
        return out
    except Exception as exc:  # the baseline must not sink the bench line
        return {"value": None, "unit": "factor-pairs/s", "cores": os.cpu_count(), "kind": "oracle",
                "sample": f"failed: {exc}"}


def run_e2e(args, g, m, data, world, rank, dev, seed, t, allreduce):
    """Same iteration through the public API with host buffers: every step's observations go H2D
    from pinned memory and its log Pe and new Q (M-step result) come back D2H.  The copies run on
    a second stream, pipelined with the compute (B200 rule: overlap copies with compute): step
    t+1's observations upload while step t's pair kernels run (the column prep is their only
    reader), and step t's results -- snapshotted on the device after its M-step -- download while
    step t+1 runs.  Every step's copies lie inside the timed region (the first upload starts after
    the start event, the end event waits for the last download)."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    cs = torch.cuda.Stream(device=dev)
    x_host = g.x.cpu().pin_memory()
    y_host = g.y.cpu().pin_memory() if g.y is not None else None
    outs = [torch.empty_like(lv["q_mean"], device="cpu").pin_memory() for lv in g.levels]
    outv = [torch.empty_like(lv["q_var"], device="cpu").pin_memory() for lv in g.levels]
    lp_host = torch.empty(1, dtype=torch.float64).pin_memory()
    h2d = x_host.numel() * x_host.element_size() + (y_host.numel() * y_host.element_size() if y_host is not None else 0)
    d2h = 8 + sum(o.numel() * 4 * 2 for o in outs)
    ev = lambda: torch.cuda.Event()  # noqa: E731

    def upload():
        with torch.cuda.stream(cs):
            g.x.copy_(x_host, non_blocking=True)
            if y_host is not None:
                g.y.copy_(y_host, non_blocking=True)
        e = ev()
        e.record(cs)
        return e

    # the step's results are snapshotted on the device (D2D, in stream order) and downloaded from the
    # snapshot, so the next step's M-step never waits for the PCIe copy of this one
    stage_lp = torch.empty_like(g.log_pe)
    stage_q = [(torch.empty_like(lv["q_mean"]), torch.empty_like(lv["q_var"])) for lv in g.levels]

    def snapshot():
        stage_lp.copy_(g.log_pe)
        for (sm, sv), lv in zip(stage_q, g.levels):
            sm.copy_(lv["q_mean"])
            sv.copy_(lv["q_var"])

    def download():
        with torch.cuda.stream(cs):
            lp_host.copy_(stage_lp, non_blocking=True)
            for o, ov, (sm, sv) in zip(outs, outv, stage_q):
                o.copy_(sm, non_blocking=True)
                ov.copy_(sv, non_blocking=True)
        e = ev()
        e.record(cs)
        return e

    # the column prep is the observations' only reader: libqem records `prep_done` on the stream right
    # after it (the forward pair kernel's start event), and the next step's upload waits for that
    prep_done = torch.cuda.Event()
    g.set_kernel_events([prep_done])

    def run(n, t, copies=True):
        if not copies:  # control: the same issue order and events, without the host copies
            x_ready, d2h_done = ev(), None
            x_ready.record(cs)
        else:
            x_ready, d2h_done = upload(), None
        for s in range(n):
            stream.wait_event(x_ready)           # this step's observations are on the device
            g.sample_estep_forward(seed, t)
            if s + 1 < n:                        # next step's upload overlaps this step's forward pair kernel
                cs.wait_event(prep_done)
                if copies:
                    x_ready = upload()
                else:
                    x_ready = ev()
                    x_ready.record(cs)
                # ... and is done before the backward: an H2D copy running under config 4's FFMA backward
                # measured 0.5 ms of slowdown, under the forward none (tools/e2e_diag.py)
                stream.wait_event(x_ready)
            allreduce()
            g.estep_backward()
            g.mstep(t)
            if d2h_done is not None:
                stream.wait_event(d2h_done)      # the previous snapshot has left the device (a step ago)
            snapshot()
            done = ev()
            done.record(stream)
            cs.wait_event(done)
            if copies:
                d2h_done = download()
            else:
                d2h_done = ev()
                d2h_done.record(cs)
            t += 1
        stream.wait_event(d2h_done)
        return t

    from paper_2503_08264_b200 import synth

    def restart():
        """Back to the main measurement's start (Q = N(0,1), m_0 = (0, 1), t = 1): the per-step cost
        depends on the regime of the run (the forward's tile modes), so the e2e loop times the same
        iterations W+1 .. W+K as the device-timed line."""
        g.set_q(synth.initial_q(m))
        g.set_state([(q, v) for q, v in synth.initial_q(m)])
        return 1

    def timed(copies):
        t = run(args.warmup, restart(), copies)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(stream)
        cs.wait_event(st)
        run(args.steps, t, copies)
        en.record(stream)
        torch.cuda.synchronize()
        return st.elapsed_time(en)

    ms = timed(True)
    ms_ctrl = timed(False)  # control: the same loop and iterations without the copies
    g.set_kernel_events(None)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
    ms_step = ms / args.steps
    return {"value": m.pairs / (ms_step * 1e-3), "unit": "factor-pairs/s", "ms_per_step": ms_step,
            "ms_per_step_same_loop_without_copies": ms_ctrl / args.steps,
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
            "overlap": "copies on a second stream: step t+1's upload under step t's forward pair kernel (after the "
                       "column prep, the observations' only reader; done before the backward); step t's results "
                       "snapshotted on the device (D2D) and downloaded under step t+1"}


def run_fresh_variant(args, m, data, dev, seed):
    """NEXT row f2: the same QEM iteration with the fresh-sample denominator
     -- an independent draw z_new, its forward + root evidence, then the E-step
    and the ratio-scaled M-step.  Device-timed like the main line, W warm-up + K steps."""
    import torch
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m, device=dev, fresh_denominator=True)
    g.set_data(data)
    stream = torch.cuda.current_stream()
    # every timed step restarts from the same Q_t (device copies): the free-running estimator's
    # ratio exp(log Pe(z) - log Pe(z_new)) overflows within a few iterations at this scale
    # (R28), and NaN states would not time the real work
    q0 = [(lv["q_mean"].clone(), lv["q_var"].clone()) for lv in g.levels]

    def one(t):
        for lv, (qm, qv) in zip(g.levels, q0):
            lv["q_mean"].copy_(qm)
            lv["q_var"].copy_(qv)
        g.sample_q(seed=seed, iter=t | (1 << 23))
        g.estep_evidence()
        g.sample_q(seed=seed, iter=t)
        g.estep()
        g.mstep(t)

    t = 1
    for _ in range(args.warmup):
        one(t)
        t += 1
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record(stream)
    for _ in range(args.steps):
        one(t)
        t += 1
    en.record(stream)
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / args.steps
    g.close()
    return {"ms_per_step": ms, "value": m.pairs / (ms * 1e-3), "unit": "factor-pairs/s (E-step pairs; the evidence "
            "pass's forward pairs are extra work)", "qem_iters_per_s": 1e3 / ms}


def run_predictive_variant(m, data, dev, seed, S=100, reps=5):
    """NEXT row f3 (R31): after an E-step of the bench workload, S = 100 backward index
    resamples ("averaged over 100 predictive samples") + the predictive
    log-likelihood of a held-out set of J observations per group; CUDA-event timed."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import QEM
    g = QEM(m, device=dev)
    g.set_data(data)
    g.set_q(synth.initial_q(m))
    g.iterate(1, 4, seed=seed)
    g.sample_q(seed=seed, iter=5)
    g.estep()
    g.set_test_data(synth.make_test_data(m, data))  # uploaded once, outside the timed region
    ir, ix = g.backward_resample(S, 1)
    g.predictive_loglik(ix)
    torch.cuda.synchronize()
    st, mid, en = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    st.record()
    for r in range(reps):
        ir, ix = g.backward_resample(S, 2 + r)
    mid.record()
    for r in range(reps):
        pll, ll_s, _ = g.predictive_loglik(ix)
    en.record()
    torch.cuda.synchronize()
    out = {"S": S, "resample_ms": st.elapsed_time(mid) / reps, "predict_ms": mid.elapsed_time(en) / reps,
           "pll": float(pll.item()), "J_test": int(m.J),
           "resampled_rows_per_s": S * m.n * m.K / (st.elapsed_time(mid) / reps * 1e-3)}
    g.close()
    return out


def run_crossed_variant(dev, steps=10):
    """NEXT row f4 (R33, R37): one QEM iteration of the Bus-shaped crossed-effects model (120
    year-borough groups, 40 journeys each, 57 companies, 6 journey types, K = 64): the K x K x J
    factor through materialised fp64 tables (CrossedQEM's default: 4 MB here) and on chip."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import CrossedQEM
    cm = synth.bus_crossed()
    out = {"workload": f"bus-crossed n={cm.n} J={cm.J} C={cm.C} T={cm.T} K={cm.K}"}
    for path, tables in (("tables", True), ("on_chip", False)):
        g = CrossedQEM(cm, device=dev, tables=tables)
        for t in range(1, 4):
            g.step(t, 3)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for t in range(4, 4 + steps):
            g.step(t, 3)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / steps
        out[path] = {"ms_per_step": ms, "pair_obs_terms_per_s": cm.n * cm.K * cm.K * cm.J / (ms * 1e-3),
                     "qem_iters_per_s": 1e3 / ms}
    return out


def run_gamma_variant(dev, steps=10):
    """NEXT row f1, Gamma / Beta Q (R32, R37): one QEM iteration of the Gamma-Poisson
    (2000 groups, J = 8, K = 128) and Beta-Binomial (2000 groups, K = 128) hierarchies, with the
    separable factors evaluated on chip (default) and through materialised fp64 tables."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import BetaBinomialQEM, GammaPoissonQEM

    def timed(make):
        g = make()
        for t in range(1, 4):
            g.step(t, 3)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for t in range(4, 4 + steps):
            g.step(t, 3)
        en.record()
        torch.cuda.synchronize()
        return st.elapsed_time(en) / steps

    gp, bb = synth.gamma_poisson(), synth.beta_binomial()
    out = {}
    for name, model, cls in (("gamma_poisson", gp, GammaPoissonQEM), ("beta_binomial", bb, BetaBinomialQEM)):
        res = {"workload": f"{name.replace('_', '-')} n={model.n} K={model.K}"}
        for path, tables in (("separable", False), ("tables", True)):
            ms = timed(lambda: cls(model, device=dev, tables=tables))
            res[path] = {"ms_per_step": ms, "factor_pairs_per_s": model.n * model.K * model.K / (ms * 1e-3),
                         "qem_iters_per_s": 1e3 / ms}
        out[name] = res
    return out


def run_qmp_variant(dev, n=20_000, K=256, J=32, steps=10):
    """NEXT row f4, second half (R43): one MPIW E-step under the non-factorised Q_MP
    (child drawn at a copy of its parent; permutation and mixture densities) on a config-4-shaped
    Gaussian hierarchy: qem_cols_qmp_gaussian -> qem_estep_separable -> qem_moments_qmp, all fp64,
    no n x K x K table; CUDA events after 3 warm-up E-steps.  Inputs drawn with torch on the device."""
    import torch
    from paper_2503_08264_b200.qem import QMP_MIXTURE, QMP_PERMUTATION, estep_qmp_gaussian
    gen = torch.Generator(device=dev).manual_seed(4)
    f32 = dict(dtype=torch.float32, device=dev)
    zt = torch.randn(n, 1, generator=gen, **f32) + 0.3
    x = zt + torch.randn(n, J, generator=gen, **f32)
    mu = 0.3 + torch.randn(K, generator=gen, **f32)
    prec = 1.0 + J
    q = torch.stack([x.sum(1).double() / prec, torch.full((n,), 0.8 / prec, dtype=torch.float64, device=dev),
                     torch.full((n,), 1.0 / prec, dtype=torch.float64, device=dev)], 1)
    eps = torch.randn(n, K, generator=gen, **f32)
    rm, rv = torch.full((1,), 0.3, **f32), torch.ones(1, **f32)
    out = {"workload": f"qmp-gaussian n={n} K={K} J={J} (fp64)"}
    for name, scheme in (("permutation", QMP_PERMUTATION), ("mixture", QMP_MIXTURE)):
        if scheme == QMP_PERMUTATION:
            copy = torch.argsort(torch.rand(n, K, generator=gen, device=dev), dim=1).to(torch.int32)
        else:
            copy = torch.randint(0, K, (n, K), generator=gen, device=dev, dtype=torch.int32)
        for _ in range(3):
            r = estep_qmp_gaussian(mu, rm, rv, q, copy, eps, x, scheme)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for _ in range(steps):
            r = estep_qmp_gaussian(mu, rm, rv, q, copy, eps, x, scheme)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / steps
        out[name] = {"ms_per_estep": ms, "factor_pairs_per_s": n * K * K / (ms * 1e-3),
                     "log_pe": float(r["log_pe"][0])}
    return out


def run_discrete_variant(dev, steps=10):
    """NEXT row f1, E-step side (R30): one QEM iteration of the Occupancy-shaped
    discrete-latent model (14400 categorical sites under a 2-d Gaussian root, K = 64; device
    Philox samples), with the factorised E-step (O(n K C)) and with materialised fp64 log-factor
    tables (O(n K^2)); CUDA events after 3 warm-up iterations."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import CategoricalQEM
    om = synth.occupancy()
    out = {"workload": f"occupancy n={om.n} C={om.C} R={om.R} d={om.d} K={om.K}"}
    for name, tables in (("factorised", False), ("tables", True)):
        g = CategoricalQEM(om, device=dev, tables=tables)
        for t in range(1, 4):
            g.step(t, 7)
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for t in range(4, 4 + steps):
            g.step(t, 7)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / steps
        out[name] = {"ms_per_step": ms, "qem_iters_per_s": 1e3 / ms,
                     "factor_pairs_per_s": om.n * om.K * om.K / (ms * 1e-3)}
        del g
    return out


def run_mstep_family_variant(dev, n=1_000_000, reps=10):
    """NEXT row f1: EMA + M-step of the non-Gaussian Q families on 1e6 latent
    instances each (Gamma / Beta Newton iterations in fp64, one thread per instance)."""
    import torch
    from paper_2503_08264_b200.qem import BETA, GAMMA, mstep_family
    g = torch.Generator(device=dev).manual_seed(0)
    out = {}
    for name, fam in (("gamma", GAMMA), ("beta", BETA)):
        a = torch.exp(torch.rand(n, 2, generator=g, device=dev, dtype=torch.float64) * 4 - 2)
        if fam == GAMMA:  # mean parameters (k/th, psi(k) - ln th) of random (k, th)
            m = torch.stack([a[:, 0] / a[:, 1], torch.special.digamma(a[:, 0]) - torch.log(a[:, 1])], 1)
        else:
            s = torch.special.digamma(a.sum(1))
            m = torch.stack([torch.special.digamma(a[:, 0]) - s, torch.special.digamma(a[:, 1]) - s], 1)
        ema = m.clone()
        mstep_family(fam, 0.7, m, ema)  # warm-up
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for _ in range(reps):
            mstep_family(fam, 0.7, m, ema)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / reps
        out[name] = {"instances": n, "ms": ms, "ns_per_instance": ms * 1e6 / n}
    return out


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) as it stands, rank 0 only.

    Each step is one oracle QEM iteration (E-step + EMA + M-step, Alg. 1) on a bounded sample of
    n_s groups of the workload, n_s sized from a probe so the W + K steps end within ~budget
    seconds; W untimed, K timed (wall clock, host)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2503_08264_b200 import synth
    full = synth.config(args.config)
    cores = os.cpu_count() or 1
    orc.set_num_threads(cores)
    budget = max(2.0, min(120.0, args.cpu_budget * 4))
    # probe: one step on `cores` groups sizes the per-step sample
    n_s = max(1, min(full.n, cores))
    m = synth.config(args.config, n=n_s)
    data, seed = synth.make_data(m), 100 + args.config
    state = orc.initial_state(m)
    q = [orc.mstep(a, b)[:2] for a, b in state]
    t0 = time.perf_counter()
    orc.qem_step(m, state, q, orc.eps_for_iteration(m, 1, seed), 1, data=data)
    probe = time.perf_counter() - t0
    per_step = budget / (args.steps + args.warmup)
    n_s = int(max(1, min(full.n, n_s * per_step / max(probe, 1e-4))))
    m = synth.config(args.config, n=n_s)
    data = synth.make_data(m)
    state = orc.initial_state(m)
    q = [orc.mstep(a, b)[:2] for a, b in state]
    times = []
    for t in range(1, args.warmup + args.steps + 1):
        eps = orc.eps_for_iteration(m, t, seed)
        t0 = time.perf_counter()
        r = orc.qem_step(m, state, q, eps, t, data=data)
        dt = time.perf_counter() - t0
        state, q = r["state"], r["q_next"]
        if t > args.warmup:
            times.append(dt)
    ms_step = 1e3 * sum(times) / len(times)
    pps = m.pairs / (ms_step * 1e-3)
    desc = (f"oracle fp64 QEM iterations (E-step + EMA + M-step) of config {args.config} on a sample of {n_s} of "
            f"{full.n} groups (K={full.K}), {args.warmup} warm-up + {args.steps} timed steps, OpenMP threads="
            f"{orc.num_threads()}")
    line = {
        "impl": "reference",
        "metric": "E-step factor-pairs/sec (N*K^2) and QEM iters/sec",
        "value": pps,
        "unit": "factor-pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "ms_per_step_basis": f"one step = the sampled {n_s}-group iteration (measured, not extrapolated)",
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (ancestral draw from the config's prior, numpy PCG64 seed = config id)",
        "qem_iters_per_s_full_workload_extrapolated": pps / full.pairs,
        "config": {"workload": f"config{args.config}:{full.name}", "M_groups": full.n, "K": full.K, "d": full.d,
                   "J": full.J, "pairs_per_step": full.pairs, "sample_groups_per_step": n_s,
                   "sample_pairs_per_step": m.pairs, "parallelism": "CPU oracle, OpenMP over groups"},
        "cpu_baseline": {"value": pps, "unit": "factor-pairs/s", "cores": orc.num_threads(), "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": pps, "unit": "factor-pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_converged_variant(args, dev, steps=5):
    """Converged-regime timing (the expm1-polynomial forward tile modes, DESIGN.md "Forward
    numerics"): configs 4 and 5 with Q near the posterior (synth.posterior_like_q); every timed step
    restarts from that Q (a device copy) so the regime holds, then sample -> E-step -> M-step.
    Reports the forward mode histogram and the forward's rate against the FMA-pipe roofline of
    the modes it ran (per pair: the d-term (FFMA) or tcgen05 contraction, the degree-n Horner
    expm1, the P-weighted accumulate; online-lse mode: one exp on the SFU)."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import QEM
    out = {}
    degs = [3, 4, 5, 7, 9]
    for cid in (4, 5):
        m = synth.config(cid)
        data = synth.make_data(m)
        g = QEM(m, device=dev)
        g.set_data(data)
        g.set_q(synth.posterior_like_q(m, data, seed=5, shrink=1.0))
        q0 = [(lv["q_mean"].clone(), lv["q_var"].clone()) for lv in g.levels]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

        def one(t):
            for lv, (qm, qv) in zip(g.levels, q0):
                lv["q_mean"].copy_(qm)
                lv["q_var"].copy_(qv)
            g.sample_q(seed=100 + cid, iter=t)
            g.estep()
            g.mstep(t)

        for t in range(1, 4):
            one(t)
        torch.cuda.synchronize()
        g.mode_hist()
        fwd = 0.0
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for t in range(4, 4 + steps):
            g.set_kernel_events(ev)
            one(t)
            torch.cuda.synchronize()
            fwd += ev[0].elapsed_time(ev[1])
        en.record()
        torch.cuda.synchronize()
        g.set_kernel_events(None)
        hist = g.mode_hist()
        fwd /= steps
        # step time without the per-step syncs: a second pass, device-timed back to back
        st.record()
        for t in range(4 + steps, 4 + 2 * steps):
            one(t)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / steps
        tot = max(1, sum(hist[:6]))  # forward modes only (slot 6: backward moment groups, 7: lazy-max redos)
        tc = g.pair_path() == 1
        base = 2.0 if tc else m.d + 2.0   # the log-factor (FFMA path) or the TMEM value (TC) per pair
        # clocks per pair per SM from the mode mix: poly mode n: (base + n + 2) FMA lane-ops / 128;
        # online mode: 1 exp / 16 (SFU) vs base + 2 FMA lane-ops
        cyc = 0.0
        for md, c in enumerate(hist[:6]):
            frac = c / tot
            if md < 5:
                cyc += frac * (base + degs[md] + 2.0) / FP32_PER_SM_CLK
            elif md == 5:
                cyc += frac * max(1.0 / SFU_PER_SM_CLK, (base + 2.0) / FP32_PER_SM_CLK)
        ceiling = SMS * SM_MAX_MHZ * 1e6 / cyc
        achieved = m.pairs / (fwd * 1e-3)
        roof = {"bound": "alu", "pipe": "fma (mode mix)", "achieved": achieved / 1e9, "peak": ceiling / 1e9,
                "unit": "Gpair/s", "frac": achieved / ceiling}
        if not tc and m.d == 1 and sum(hist[:5]) > 0:
            # d = 1 Taylor modes run as moment tiles (R38): no per-pair work, so the per-pair
            # mode-mix ceiling is a reference line, not a roofline of what runs
            roof = {"bound": "fp64 (moment tiles, DESIGN.md R38)", "unit": "Gpair/s", "achieved": achieved / 1e9,
                    "pairwise_mode_mix_ceiling": ceiling / 1e9, "over_pairwise_ceiling": achieved / ceiling}
        out[f"config{cid}"] = {"ms_per_step": ms, "qem_iters_per_s": 1e3 / ms, "value": m.pairs / (ms * 1e-3),
                               "unit": "factor-pairs/s", "forward_ms": fwd,
                               "forward_mode_hist": {"expm1_deg3": hist[0], "deg4": hist[1], "deg5": hist[2],
                                                     "deg7": hist[3], "deg9": hist[4], "online_lse": hist[5]},
                               "backward_moment_groups": hist[6],
                               "forward_roofline": roof}
        g.close()
    return out


def run_iterate_variant(dev):
    """QEM iterations/s of every config through qem_iterate's captured CUDA graph (the library's own
    loop: Philox sampler -> E-step -> EMA/M-step), device-timed after 5 warm-up iterations."""
    import torch
    from paper_2503_08264_b200 import synth
    from paper_2503_08264_b200.qem import QEM
    out = {}
    for cid in (1, 2, 3, 4, 5):
        m = synth.config(cid)
        T = 200 if cid <= 3 else 10
        g = QEM(m, device=dev, trace_len=T)
        g.set_data(synth.make_data(m))
        g.set_q(synth.initial_q(m))
        g.iterate(1, 5, seed=100 + cid, use_graph=True)
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        g.iterate(6, T, seed=100 + cid, use_graph=True)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / T
        out[f"config{cid}"] = {"us_per_iteration": ms * 1e3, "qem_iters_per_s": 1e3 / ms,
                               "factor_pairs_per_s": m.pairs / (ms * 1e-3), "iterations": f"6..{5 + T}",
                               "kernels_per_iteration": g.kernel_launches() // T}
        g.close()
    return out


def _relaunch_torchrun(n: int) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run, one rank per GPU."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init log (nranks, transport) stays on ...
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout carries the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="qem", choices=["qem", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
