#!/usr/bin/env python3
"""bench.py -- one JSON line: varying-parameter deviates on B200 (BASELINE.json).

A STEP is one pass of the whole hot path over the five
BASELINE.json configs at full size:
  cfg1  Gibbs 1024 chains x 1000 sweeps, all samples stored          (K5-K7)
  cfg2  varying-parameter Gaussian + uniform fills, 2^28 f32 each     (K2)
  cfg3  varying-alpha Gamma, 2^26 f64                                 (K3)
  cfg4  LDA-shaped Dirichlet 10^6 x 256 f32                           (K4)
  cfg5  Gibbs 2^24 chains x 4096 sweeps, per-chain stats + histogram (K5-K7)
        + the NCCL all-reduce of the totals when N > 1
A sample is one output deviate (Gibbs: one conditional draw, 2 per sweep;
Dirichlet: one component).  value = all samples of the job / max-over-ranks
device time.

--scaling strong (default, BASELINE configs[3]/[4]
"documents/chains sharded across GPUs"): the configs keep their totals and
rank r draws its contiguous shard of every config's units at the counters
that shard has in the 1-GPU run (paper_1412_4825_b200/shard.py), so the union
over ranks is bit for bit the 1-GPU step.  At N > 1 a secondary weak-scaling
run (every rank the full configs on a disjoint counter range) is reported
under "weak".  --scaling weak makes that the headline.

--impl reference times the CPU oracle (oracle/, the reference arm of this
tier) on bounded samples of the same workload on the host cores.
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

METRIC = "Gsamples/s varying-param Gamma & Gibbs at 1/2/4/8 B200; % of roofline"
UNIT = "Gsamples/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0          # B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 8000.0           # BASELINE north_star "roughly 8 TB/s" (report both)
SMS, SMSP, LANES = 148, 4, 32
# Gibbs roofline: the sweep is bound by the B200
# FMA-heavy pipe, which runs every fp64 op (64 lanes/clk/SM) and the 32x32->64
# IMAD.WIDE of Philox at half that rate (tools/ubench.cu, profiles/).  The
# algorithmic per-chain work of one sweep is 16 wide multiplies (20 Philox
# products minus the 3 that are constant along a chain and the round-2 M1
# product, which depends only on the sweep and is computed once per sweep
# for all chains) + 9 fp64 ops (2 x (1-y, mul), 5 statistics)
# = 16*2 + 9 = 41 fp64-pipe slots; peak = 64 x 148 x f_sm.
GIBBS_PIPE_OPS_PER_SWEEP = 41
FP64_LANES_PER_SM = 64
# cfg1 (1024 chains) is LATENCY-bound: a chain's sweeps are serial and each
# sweep's critical path is 4 dependent fp64 ops (fma, mul, fma, mul) at the
# measured 8.1-cycle dependent latency (tools/ulat.cu, profiles/) = 32.1
# cycles/sweep; floor = n_sweeps x 32.1 / f_sm for any number of chains that
# fits one wave.
GIBBS_SWEEP_LATENCY_CYC = 32.1
# Gamma / Dirichlet roofline (DESIGN.md §7 K3): the same FMA-heavy pipe as
# Gibbs.  Algorithmic slots of the method as implemented (fp64 ops + 2 per
# IMAD.WIDE), counted from the kernel's arithmetic:
#   trial = Philox 19 IMAD.WIDE (38) + 1-u53 1 + ln 14 + sqrt 7 + cos 13
#           + d, c 8 + cz, t, v, g 5 + z, -2L 2                      = 88
#   boost = Philox 38 + 1-u53 1 + ln 14 + divide 8 + exp 11 + 2 mul = 74
#   sample: x beta (Gamma) or x 1/S + sum (Dirichlet)                = 1 / 2
# evaluated on the measured trial / boost mix of each config.
# SURVEY.md §8(d)'s issue model: ~68 issue slots per Gibbs sweep (Philox 40,
# 2 u53 ~12, 4 fp64 update, 4 stats, bin + ATOMS ~5, loop ~3); Gamma ~195
# and Dirichlet ~270 slots per sample, against 148 x 4 x 32 lanes x f_sm.
GIBBS_ISSUE_SLOTS_PER_SWEEP = 68
GAMMA_ISSUE_SLOTS_SURVEY = {"cfg3_gamma": 195, "cfg4_dirichlet": 270}
GAMMA_TRIAL_SLOTS = 88
GAMMA_BOOST_SLOTS = 74
GAMMA_SAMPLE_SLOTS = 1
DIRICHLET_SAMPLE_SLOTS = 2


def _ncu_entry(kernel_substr):
    """The newest committed ncu --set full summary (profiles/*_ncu.json,
    tools/ncu_summary.py) entry of a kernel: the full-size launch, i.e. the
    longest capture of that kernel in the newest file that has one (a file
    may also hold a smaller launch of the same kernel, e.g. a strong-scaling
    shard)."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu.json"))):
        try:
            with open(path) as f:
                ks = [k for k in json.load(f)["kernels"] if kernel_substr in k.get("kernel", "")]
        except Exception:
            continue
        if ks:
            best = (max(ks, key=lambda k: k.get("time_ms", 0.0)), os.path.basename(path))
    return best


def ncu_traffic(kernel_substr):
    """DRAM bytes (read + write) per launch of a kernel from the committed ncu
    summary, or None."""
    e = _ncu_entry(kernel_substr)
    if e is None or "traffic_GB" not in e[0]:
        return None
    return e[0]["traffic_GB"] * 1e9, e[1]


NCU_KERNEL = {"cfg1_gibbs": "gibbs_lat_kernel<1>", "cfg2_gaussian": "fill_kernel<float, 3, 0>",
              "cfg2_uniform": "fill_kernel<float, 2, 0>", "cfg3_gamma": "gamma_kernel<double>",
              "cfg4_dirichlet": "dirichlet_smem_kernel<float>",
              "cfg5_gibbs": "gibbs_kernel<0, 3, 256, 1>"}


def ncu_evidence(kernel_substr):
    """Pipe / issue / DRAM utilisation of a kernel from the committed ncu
    summary (profiles/*_ncu.json), labelled with its file; {} if absent."""
    e = _ncu_entry(kernel_substr)
    if e is None:
        return {}
    ev = {m: e[0][m] for m in ("issue_active_pct", "fmaheavy_pct", "alu_pct", "dram_pct_peak",
                               "warps_active_pct") if m in e[0]}
    ev["source"] = e[1]
    return ev


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, 1965.0, "fallback"


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
class Workload:
    """Inputs resident in HBM, outputs preallocated, one handle per config.

    mode "strong" (default): every config keeps its BASELINE total and rank r
    draws the contiguous shard [lo, hi) of its units (paper_1412_4825_b200/
    shard.py): cfg1/cfg5 chain ranges (stream = first chain), cfg2 sample
    ranges on Philox-block boundaries, cfg3 sample ranges, cfg4 document
    ranges, each at the cursor its first unit has in the unsharded call -- so
    the union over ranks is bit for bit the 1-GPU step.  mode "weak": every
    rank runs the full configs on a disjoint counter range (rank r's Gibbs
    streams start at r * n_chains, its fill/Gamma/Dirichlet cursors r spans
    further), i.e. the samples of an N-times larger run."""

    def __init__(self, rank, world, torch, B, small=False, mode="strong"):
        import workloads as W
        from paper_1412_4825_b200 import shard as S
        self.torch, self.B, self.rank, self.world, self.mode = torch, B, rank, world, mode
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.c1, self.c2, self.c3, self.c4, self.c5 = (dict(W.CFG1), dict(W.CFG2), dict(W.CFG3),
                                                      dict(W.CFG4), dict(W.CFG5))
        if small:   # quick functional run (--small): not a bench number
            self.c2["n"] >>= 6; self.c3["n"] >>= 6; self.c4["n_docs"] //= 64
            self.c5["n_chains"] >>= 6
        f32, f64 = torch.float32, torch.float64
        N2, N3 = self.c2["n"], self.c3["n"]
        D, K = self.c4["n_docs"], self.c4["k"]
        NC5, ns5 = self.c5["n_chains"], self.c5["n_sweeps"]
        NC1, ns1 = self.c1["n_chains"], self.c1["n_sweeps"]
        if mode == "strong":
            r, w = rank, world
            self.sh1 = S.shard_range(NC1, r, w)
            self.sh2 = S.shard_range(N2, r, w, align=4)          # f32 fills: 4 per block
            self.sh3 = S.shard_range(N3, r, w)
            self.sh4 = S.shard_range(D, r, w)
            self.sh5 = S.shard_range(NC5, r, w)
        else:
            self.sh1, self.sh2, self.sh3 = (0, NC1), (0, N2), (0, N3)
            self.sh4, self.sh5 = (0, D), (0, NC5)
        nc1 = self.sh1[1] - self.sh1[0]
        n2 = self.sh2[1] - self.sh2[0]
        n3 = self.sh3[1] - self.sh3[0]
        d4 = self.sh4[1] - self.sh4[0]
        nc5 = self.sh5[1] - self.sh5[0]
        self.n1, self.n2, self.n3, self.d4, self.n5 = nc1, n2, n3, d4, nc5

        def part(full, lo, hi):
            # the shard's slice of the full parameter arrays (identical bytes to
            # the unsharded run's), materialised alone
            if (lo, hi) == (0, full.shape[0]):
                return full
            return full[lo:hi].clone()
        p2 = W.cfg2_params(N2, seed=self.c2["seed"], device=dev)
        self.p2 = {k: part(v, *self.sh2) for k, v in p2.items()}
        del p2
        p3 = W.cfg3_params(N3, seed=self.c3["seed"], device=dev)
        self.p3 = {k: part(v, *self.sh3) for k, v in p3.items()}
        del p3
        self.p4 = part(W.cfg4_params(D, K, seed=self.c4["seed"], device=dev), *self.sh4)
        torch.cuda.empty_cache()
        self.o2g = torch.empty(n2, dtype=f32, device=dev)
        self.o2u = torch.empty(n2, dtype=f32, device=dev)
        self.o3 = torch.empty(n3, dtype=f64, device=dev)
        self.o4 = torch.empty(d4, K, dtype=f32, device=dev)
        self.o1x = torch.empty(ns1, nc1, dtype=f64, device=dev)
        self.o1y = torch.empty(ns1, nc1, dtype=f64, device=dev)
        self.st5 = torch.empty(5, nc5, dtype=f64, device=dev)
        self.fx5 = torch.empty(2, nc5, dtype=f64, device=dev)
        self.tot5 = torch.empty(B.TOTALS_LEN, dtype=f64, device=dev)
        self.tot1 = torch.empty(B.TOTALS_LEN, dtype=f64, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        if mode == "strong":
            self.h1 = B.brng_create(self.c1["seed"], S.gibbs_stream(0, self.sh1[0]))
            self.h5 = B.brng_create(self.c5["seed"], S.gibbs_stream(0, self.sh5[0]))
            self.base2 = S.fill_cursor(0, self.sh2[0], 4)
            self.base3 = S.gamma_cursor(0, self.sh3[0])
            self.base4 = S.dirichlet_cursor(0, self.sh4[0], K)
        else:
            self.h1 = B.brng_create(self.c1["seed"], rank * NC1)
            self.h5 = B.brng_create(self.c5["seed"], rank * NC5)
            self.base2 = rank * 2 * ((N2 + 3) // 4)
            self.base3 = rank * 256 * N3
            self.base4 = rank * 256 * D * K
        self.h2 = B.brng_create(self.c2["seed"], 0)
        self.h3 = B.brng_create(self.c3["seed"], 0)
        self.h4 = B.brng_create(self.c4["seed"], 0)
        for h in (self.h1, self.h2, self.h3, self.h4, self.h5):
            B.brng_set_cuda_stream(h, s)
        self.samples = {
            "cfg1_gibbs": 2 * nc1 * ns1, "cfg2_gaussian": n2, "cfg2_uniform": n2,
            "cfg3_gamma": n3, "cfg4_dirichlet": d4 * K, "cfg5_gibbs": 2 * nc5 * ns5,
        }
        # samples of the whole job (all ranks): the configs' totals (strong) or
        # N times this rank's (weak)
        full = {"cfg1_gibbs": 2 * NC1 * ns1, "cfg2_gaussian": N2, "cfg2_uniform": N2,
                "cfg3_gamma": N3, "cfg4_dirichlet": D * K, "cfg5_gibbs": 2 * NC5 * ns5}
        self.job_samples = sum(full.values()) * (1 if mode == "strong" else world)
        self.names = list(self.samples)
        # our kernels per step: cfg1 gibbs + K7, 2 fills, Gamma, Dirichlet,
        # cfg5 gibbs + K7
        self.launches_per_step = 8
        self.trials = None

    def reset_cursors(self):
        B = self.B
        B.brng_set_offset(self.h1, 0); B.brng_set_offset(self.h2, self.base2)
        B.brng_set_offset(self.h3, self.base3); B.brng_set_offset(self.h4, self.base4)
        B.brng_set_offset(self.h5, 0)

    def step(self, ev=None, allreduce=None):
        """Enqueue one step; ev: dict name -> (start, end) events to record."""
        B, torch = self.B, self.torch
        self.reset_cursors()
        n2, n3 = self.n2, self.n3
        D, K = self.d4, self.c4["k"]

        def run(name, fn):
            if ev is not None:
                ev[name][0].record()
            fn()
            if ev is not None:
                ev[name][1].record()

        run("cfg1_gibbs", lambda: B.brng_gibbs_triangle(
            self.h1, self.n1, self.c1["n_sweeps"], None, None, 0, self.o1x,
            self.o1y, None, None, self.tot1))
        run("cfg2_gaussian", lambda: B.brng_gaussian_f32(self.h2, self.p2["mu"], self.p2["sigma"],
                                                         self.o2g, n2))
        run("cfg2_uniform", lambda: B.brng_uniform_f32(self.h2, self.p2["a"], self.p2["b"],
                                                       self.o2u, n2))
        run("cfg3_gamma", lambda: B.brng_gamma_f64(self.h3, self.p3["alpha"], self.p3["beta"],
                                                   self.o3, n3, self.trials))
        run("cfg4_dirichlet", lambda: B.brng_dirichlet_f32(self.h4, self.p4, D, K, self.o4, None))
        run("cfg5_gibbs", lambda: B.brng_gibbs_triangle(
            self.h5, self.n5, self.c5["n_sweeps"], None, None, 0, None, None,
            self.st5, self.fx5, self.tot5))
        if allreduce is not None:
            if ev is not None and "nccl_totals" in ev:
                run("nccl_totals", lambda: allreduce(self.tot5))
            else:
                allreduce(self.tot5)

    def checksums(self):
        """Bit-level checksums of every output of a step (sum of the raw 32-bit
        words, exact), to show the step is deterministic across repetitions."""
        torch = self.torch
        outs = {"cfg1_gibbs": (self.o1x, self.o1y, self.tot1), "cfg2_gaussian": (self.o2g,),
                "cfg2_uniform": (self.o2u,), "cfg3_gamma": (self.o3,),
                "cfg4_dirichlet": (self.o4,), "cfg5_gibbs": (self.st5, self.fx5, self.tot5)}
        res = {}
        for name, ts in outs.items():
            h = 0
            for t in ts:
                h = (h * 1000003 + int(t.contiguous().view(torch.int32).to(torch.int64).sum()
                                       .item())) % (1 << 61)
            res[name] = h
        return res

    def destroy(self):
        for h in (self.h1, self.h2, self.h3, self.h4, self.h5):
            self.B.brng_destroy(h)


def timed_steps(wl, torch, dist, world, local, steps, warmup, allreduce):
    """W untimed warm-up steps, then K steps timed with CUDA events on the
    launching stream, bracketed by barrier + synchronize; max over ranks.
    Returns ms per step, per-row median device times, per-step times, clocks
    sampled during the timed region, and the per-step events."""
    for _ in range(warmup):
        wl.step(allreduce=allreduce)
    torch.cuda.synchronize()
    names = wl.names
    ev_names = list(names) + (["nccl_totals"] if world > 1 else [])
    evs = [{n: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for n in ev_names} for _ in range(steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    t0.record()
    marks[0].record()
    for k in range(steps):
        wl.step(ev=evs[k], allreduce=allreduce)
        marks[k + 1].record()
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
    step_ms = [marks[k].elapsed_time(marks[k + 1]) for k in range(steps)]
    # per-row device times: median over the timed steps
    per = {n: statistics.median(e[n][0].elapsed_time(e[n][1]) for e in evs) for n in names}
    return ms / steps, per, step_ms, clk, evs


def roofline_models(n_sweeps_units, t_s, sm_hz):
    """Gibbs (cfg5) against both rooflines: the FMA-heavy-pipe model that binds
     and SURVEY.md §8(d)'s issue model, each with its slot count
    and peak spelled out so frac can be recomputed from the line alone."""
    pipe_peak = SMS * FP64_LANES_PER_SM * sm_hz
    issue_peak = SMS * SMSP * LANES * sm_hz
    pipe = GIBBS_PIPE_OPS_PER_SWEEP * n_sweeps_units / t_s
    issue = GIBBS_ISSUE_SLOTS_PER_SWEEP * n_sweeps_units / t_s
    return {
        "pipe": {"slots_per_sweep": GIBBS_PIPE_OPS_PER_SWEEP,
                 "peak_per_s": pipe_peak, "achieved_per_s": pipe,
                 "frac": round(pipe / pipe_peak, 4),
                 "peak_formula": "148 SM x 64 fp64-pipe lanes/clk x sm clock (IMAD.WIDE = 2 "
                                 "slots; tools/ubench.cu: 62 DFMA/clk/SM)"},
        "issue_survey_8d": {"slots_per_sweep": GIBBS_ISSUE_SLOTS_PER_SWEEP,
                            "peak_per_s": issue_peak, "achieved_per_s": issue,
                            "frac": round(issue / issue_peak, 4),
                            "peak_formula": "148 SM x 4 SMSP x 32 lanes x sm clock "
                                            "(SURVEY.md §8(d): ~68 issue slots per sweep)"},
    }


def gamma_models(mt, fb, per_sample, samples, t_s, sm_hz):
    """Gamma / Dirichlet against the pipe model (DESIGN.md §7 K3) and the
    SURVEY §8(d) issue estimates (~195 slots/sample cfg3, ~270 cfg4)."""
    pipe_peak = SMS * FP64_LANES_PER_SM * sm_hz
    issue_peak = SMS * SMSP * LANES * sm_hz
    slots = mt * GAMMA_TRIAL_SLOTS + fb * GAMMA_BOOST_SLOTS + per_sample
    return slots, round(slots * samples / t_s / pipe_peak, 4), issue_peak


def gpu_arm(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # plumbing check only (tests/tools): BRNG_BENCH_DEVICE pins every rank to
    # one GPU and BRNG_BENCH_BACKEND=gloo replaces NCCL, so the N>1 code path
    # runs on a 1-GPU box (independent processes, nothing waits on a peer
    # kernel); numbers from such a run are not bench values
    local = int(os.environ.get("BRNG_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BRNG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_1412_4825_b200 as B

    hbm_peak, sm_max_cfg, peak_kind = load_peaks()
    wl = Workload(rank, world, torch, B, small=args.small, mode=args.scaling)
    allreduce = (lambda t: dist.all_reduce(t)) if world > 1 else None
    names = wl.names
    ms_step, per, step_ms, clk, evs = timed_steps(wl, torch, dist, world, local, args.steps,
                                                  args.warmup, allreduce)
    # determinism: the outputs of the last timed step vs one more (untimed) step
    # (cfg5 totals include the all-reduce, so they are compared at N = 1 only)
    cs_a = wl.checksums()
    wl.step(allreduce=allreduce)
    torch.cuda.synchronize()
    cs_b = wl.checksums()
    determinism = {"identical_across_steps": all(cs_a[k] == cs_b[k] for k in cs_a
                                                 if world == 1 or k != "cfg5_gibbs"),
                   "checksums": {k: f"{v:016x}" for k, v in cs_a.items()}}
    value = wl.job_samples / (ms_step * 1e-3) / 1e9
    errs = sum(B.brng_device_errors(h) for h in (wl.h1, wl.h2, wl.h3, wl.h4, wl.h5))

    # ---- roofline of the dominant kernel + breakdown -------------------------
    sm_hz = (clk.get("sm_max_mhz") or sm_max_cfg) * 1e6
    pipe_peak = SMS * FP64_LANES_PER_SM * sm_hz        # fp64-pipe slots / s
    # Gamma / Dirichlet trial mixes, measured once (untimed) from the trials outputs
    wl.trials = torch.empty(wl.n3, dtype=torch.uint8, device=wl.dev)
    B.brng_set_offset(wl.h3, wl.base3)
    B.brng_gamma_f64(wl.h3, wl.p3["alpha"], wl.p3["beta"], wl.o3, wl.n3, wl.trials)
    mix = {"cfg3_gamma": (wl.trials.double().mean().item(),
                          (wl.p3["alpha"] < 1).double().mean().item(), GAMMA_SAMPLE_SLOTS)}
    D4, K4 = wl.p4.shape
    wl.trials = torch.empty(D4, K4, dtype=torch.uint8, device=wl.dev)
    B.brng_set_offset(wl.h4, wl.base4)
    B.brng_dirichlet_f32(wl.h4, wl.p4, D4, K4, wl.o4, wl.trials)
    mix["cfg4_dirichlet"] = (wl.trials.double().mean().item(),
                             (wl.p4 < 1).double().mean().item(), DIRICHLET_SAMPLE_SLOTS)
    wl.trials = None
    torch.cuda.synchronize()
    bd = {}
    for n in names:
        t = per[n] * 1e-3
        d = {"ms": round(per[n], 4), "Gsamples_per_s": round(wl.samples[n] / t / 1e9, 3)}
        if n in ("cfg2_gaussian", "cfg2_uniform"):
            gbs = 12.0 * wl.samples[n] / t / 1e9
            d.update(bound="hbm", GB_per_s=round(gbs, 1), frac=round(gbs / hbm_peak, 4),
                     frac_nominal_8TBs=round(gbs / NOMINAL_HBM_GBS, 4))
        elif n in mix:
            mt, fb, per_sample = mix[n]
            slots, frac, issue_peak = gamma_models(mt, fb, per_sample, wl.samples[n], t, sm_hz)
            est = GAMMA_ISSUE_SLOTS_SURVEY[n]
            d.update(bound="alu", frac=frac, mean_trials=round(mt, 5),
                     boost_frac=round(fb, 4), pipe_slots_per_sample=round(slots, 2),
                     frac_issue_survey_8d=round(est * wl.samples[n] / t / issue_peak, 4),
                     issue_slots_per_sample_survey_8d=est)
        elif n == "cfg1_gibbs":
            floor_s = wl.c1["n_sweeps"] * GIBBS_SWEEP_LATENCY_CYC / sm_hz
            d.update(bound="latency", frac=round(floor_s / t, 4),
                     floor_us=round(floor_s * 1e6, 2),
                     Gsweeps_per_s=round(wl.samples[n] / 2 / t / 1e9, 3))
        elif n == "cfg5_gibbs":
            m = roofline_models(wl.samples[n] / 2, t, sm_hz)
            d.update(bound="alu", frac=m["pipe"]["frac"],
                     frac_issue_survey_8d=m["issue_survey_8d"]["frac"],
                     Gsweeps_per_s=round(wl.samples[n] / 2 / t / 1e9, 3))
        ev = ncu_evidence(NCU_KERNEL.get(n, "?"))
        if ev:
            d["ncu"] = ev
        bd[n] = d
    if world > 1:     # the one data-path collective (cfg5 totals, 272 doubles)
        bd["nccl_totals"] = {"ms": round(statistics.mean(
            e["nccl_totals"][0].elapsed_time(e["nccl_totals"][1]) for e in evs), 4),
            "what": "all_reduce of the cfg5 totals (272 f64) after the Gibbs kernel",
            "cfg5_with_nccl_ms": None}
        bd["nccl_totals"]["cfg5_with_nccl_ms"] = round(per["cfg5_gibbs"] +
                                                       bd["nccl_totals"]["ms"], 4)
    dom = max(names, key=lambda n: per[n])
    t_dom = per[dom] * 1e-3
    if dom in ("cfg1_gibbs", "cfg5_gibbs"):
        m = roofline_models(wl.samples[dom] / 2, t_dom, sm_hz)
        roof = {"kernel": "gibbs_kernel (" + dom + ")", "bound": "alu",
                "achieved": round(m["pipe"]["achieved_per_s"] / 1e12, 3),
                "peak": round(m["pipe"]["peak_per_s"] / 1e12, 3),
                "unit": "T fp64-pipe ops/s (FMA-heavy pipe: 64 lanes/clk/SM x 148 SM x "
                        "sm_max clock; IMAD.WIDE = 2 slots)",
                "frac": m["pipe"]["frac"],
                "algorithmic_per_unit": f"{GIBBS_PIPE_OPS_PER_SWEEP} pipe slots/sweep "
                                        "(16 per-chain IMAD.WIDE x 2 + 9 fp64)",
                "units_per_launch": wl.samples[dom] // 2,
                "sm_hz": sm_hz,
                "models": {k: {kk: (round(vv / 1e12, 4) if kk.endswith("per_s") else vv)
                               for kk, vv in v.items()} for k, v in m.items()},
                "models_unit": "per_s fields in T slots/s; frac = achieved / peak; achieved = "
                               "slots_per_sweep x units_per_launch / kernel seconds",
                "traffic": None,
                "peak_source": "derived (DESIGN.md §7): 64 fp64 lanes/clk/SM (tools/ubench.cu "
                               "measures 62 DFMA/clk/SM) x 148 SMs x the sampled sm_max clock"}
        tr = ncu_traffic(NCU_KERNEL["cfg5_gibbs"])
        if tr is not None:
            roof["traffic"] = int(tr[0])
            roof["traffic_source"] = tr[1] + " (ncu --set full, dram__bytes_read+write per "\
                "launch; algorithmic = chain_stats + final_xy writes 0.94 GB)"
    else:
        roof = {"kernel": dom, "bound": bd[dom].get("bound"), "frac": bd[dom].get("frac"),
                "peak_source": peak_kind}
    roof["hbm_peak_source"] = f"{peak_kind} ({hbm_peak:.1f} GB/s, MEASURED_PEAKS.json; fills)"

    # ---- end to end through the C ABI with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(wl, torch, B, args, allreduce, world, dist)
    wl_launches = wl.launches_per_step
    wl.destroy()
    del wl
    torch.cuda.empty_cache()

    # ---- secondary: weak scaling (every rank the full configs) ---------------
    weak = None
    if world > 1 and args.scaling == "strong" and not args.no_weak:
        wk = Workload(rank, world, torch, B, small=args.small, mode="weak")
        wms, wper, _, _, _ = timed_steps(wk, torch, dist, world, local, args.steps,
                                         args.warmup, allreduce)
        weak = {"value": round(wk.job_samples / (wms * 1e-3) / 1e9, 3), "unit": UNIT,
                "ms_per_step": round(wms, 3), "n_gpus": world,
                "what": "every rank runs the full configs on a disjoint counter range "
                        "(an N-times larger job); same timing rules",
                "cfg5_ms": round(wper["cfg5_gibbs"], 4)}
        wk.destroy()
        del wk
        torch.cuda.empty_cache()

    g3, g5 = bd["cfg3_gamma"], bd["cfg5_gibbs"]
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": step_config(world, args.small, args.scaling),
        "gamma_cfg3": {"Gsamples_per_s": g3["Gsamples_per_s"], "ms": g3["ms"],
                       "frac_pipe": g3["frac"], "frac_issue_survey_8d": g3["frac_issue_survey_8d"]},
        "gibbs_cfg5": {"Gsamples_per_s": g5["Gsamples_per_s"], "Gsweeps_per_s": g5["Gsweeps_per_s"],
                       "ms": g5["ms"], "frac_pipe": g5["frac"],
                       "frac_issue_survey_8d": g5["frac_issue_survey_8d"]},
        "roofline": roof,
        "breakdown": bd,
        "step_ms": {"median": round(statistics.median(step_ms), 3),
                    "best": round(min(step_ms), 3), "worst": round(max(step_ms), 3),
                    "note": "this rank's per-step device times; value uses the mean over "
                            "all steps, max over ranks"},
        "determinism": determinism,
        "gpu_launches": wl_launches * args.steps,
        "device_errors": errs,
        "clocks": clk,
    }
    if weak is not None:
        out["weak"] = weak
    if e2e is not None:
        out["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_run(wl, torch, B, args, allreduce, world, dist):
    """Same step through the C ABI with HOST (pinned) buffers: the library
    stages host->device, runs the kernels, copies results back (include/brng.h)."""
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hp2 = {k: pin(v) for k, v in wl.p2.items()}
    hp3 = {k: pin(v) for k, v in wl.p3.items()}
    hp4 = pin(wl.p4)
    o2g, o2u = torch.empty_like(hp2["mu"]).pin_memory(), torch.empty_like(hp2["mu"]).pin_memory()
    o3 = torch.empty_like(hp3["alpha"]).pin_memory()
    o4 = torch.empty_like(hp4).pin_memory()
    c1, c5 = wl.c1, wl.c5
    o1x = torch.empty(c1["n_sweeps"], wl.n1, dtype=torch.float64).pin_memory()
    o1y = torch.empty_like(o1x).pin_memory()
    st5 = torch.empty(5, wl.n5, dtype=torch.float64).pin_memory()
    fx5 = torch.empty(2, wl.n5, dtype=torch.float64).pin_memory()
    tot5 = torch.empty(B.TOTALS_LEN, dtype=torch.float64).pin_memory()
    tot1 = torch.empty(B.TOTALS_LEN, dtype=torch.float64).pin_memory()
    n2, n3 = wl.n2, wl.n3
    D, K = wl.d4, wl.c4["k"]

    def group_gibbs():          # compute-heavy, little I/O
        B.brng_set_offset(wl.h1, 0)
        B.brng_set_offset(wl.h5, 0)
        B.brng_gibbs_triangle(wl.h1, wl.n1, c1["n_sweeps"], None, None, 0, o1x, o1y,
                              None, None, tot1)
        B.brng_gibbs_triangle(wl.h5, wl.n5, c5["n_sweeps"], None, None, 0, None, None,
                              st5, fx5, tot5)

    def group_io():             # PCIe-heavy, short kernels
        B.brng_set_offset(wl.h2, wl.base2)
        B.brng_set_offset(wl.h3, wl.base3)
        B.brng_set_offset(wl.h4, wl.base4)
        B.brng_gaussian_f32(wl.h2, hp2["mu"], hp2["sigma"], o2g, n2)
        B.brng_uniform_f32(wl.h2, hp2["a"], hp2["b"], o2u, n2)
        B.brng_gamma_f64(wl.h3, hp3["alpha"], hp3["beta"], o3, n3, None)
        B.brng_dirichlet_f32(wl.h4, hp4, D, K, o4, None)

    def reduce():
        if allreduce is not None:
            t = tot5.to(wl.dev)
            allreduce(t)
            tot5.copy_(t.cpu())

    # the two groups are independent rows of the step: a user overlaps them by
    # calling the C ABI from two host threads with handles on two CUDA streams
    # (ctypes releases the GIL), so PCIe traffic hides under the Gibbs compute
    # the I/O rows' short kernels get the higher stream priority so they are
    # scheduled at the boundaries of the (chunked) Gibbs launches
    s_a, s_b = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
    for h in (wl.h1, wl.h5):
        B.brng_set_cuda_stream(h, s_a.cuda_stream)
    for h in (wl.h2, wl.h3, wl.h4):
        B.brng_set_cuda_stream(h, s_b.cuda_stream)

    def step_concurrent():
        err = []

        def run_gibbs():
            try:
                group_gibbs()
            except BaseException as e:          # re-raised below: no silent e2e number
                err.append(e)
        ta = threading.Thread(target=run_gibbs)
        ta.start()
        try:
            group_io()
        finally:
            ta.join()
        if err:
            raise err[0]
        reduce()

    def step_serial():
        group_gibbs()
        group_io()
        reduce()

    def timed(fn, steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        return ms

    step_serial()            # warm the staging buffers and copy streams
    step_concurrent()
    steps = max(1, args.steps if args.e2e_steps is None else args.e2e_steps)
    ms = timed(step_concurrent, steps)
    ms_serial = timed(step_serial, 1)
    ms_gibbs_rows = timed(group_gibbs, 1)       # each row group alone, for the overlap
    ms_io_rows = timed(group_io, 1)             # accounting (not part of the value)
    s0 = torch.cuda.current_stream().cuda_stream
    for h in (wl.h1, wl.h2, wl.h3, wl.h4, wl.h5):
        B.brng_set_cuda_stream(h, s0)
    h2d = 4 * n2 * 4 + 2 * n3 * 8 + D * K * 4
    d2h = 2 * n2 * 4 + n3 * 8 + D * K * 4 + 2 * wl.n1 * c1["n_sweeps"] * 8 + \
        7 * wl.n5 * 8 + 2 * B.TOTALS_LEN * 8
    total = wl.job_samples
    return {"value": round(total / (ms / steps * 1e-3) / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "ms_per_step": round(ms / steps, 3),
            "timing": "wall clock (perf_counter) between device synchronizations, max over ranks",
            "schedule": "two host threads: Gibbs rows on one CUDA stream, fill/Gamma/Dirichlet "
                        "rows (host-staged, chunk-pipelined) on a higher-priority stream",
            "serial_ms_per_step": round(ms_serial, 3),
            "gibbs_rows_alone_ms": round(ms_gibbs_rows, 3),
            "io_rows_alone_ms": round(ms_io_rows, 3)}


# ----------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ----------------------------------------------------------------------------
def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def full_units():
    """Units of each config in one full step (chains, samples, documents)."""
    import workloads as W
    return {"cfg1_gibbs": W.CFG1["n_chains"], "cfg2_gaussian": W.CFG2["n"],
            "cfg2_uniform": W.CFG2["n"], "cfg3_gamma": W.CFG3["n"],
            "cfg4_dirichlet": W.CFG4["n_docs"], "cfg5_gibbs": W.CFG5["n_chains"]}


def samples_per_unit():
    import workloads as W
    return {"cfg1_gibbs": 2 * W.CFG1["n_sweeps"], "cfg2_gaussian": 1, "cfg2_uniform": 1,
            "cfg3_gamma": 1, "cfg4_dirichlet": W.CFG4["k"], "cfg5_gibbs": 2 * W.CFG5["n_sweeps"]}


def oracle_run(units, threads, stride5=1, inputs=None):
    """Run the oracle, as it stands, over `units[name]` units of each config on
    `threads` Python threads (disjoint slices; ctypes releases the GIL).
    Parameters follow each config's recipe (workloads/, generated at that size,
    untimed).  cfg5 runs chains 0, stride5, 2*stride5, ... in blocks of 64
    consecutive chains (a stride subset of the 2^24 chains).  Returns
    {name: (units, samples, seconds)}."""
    import numpy as np
    import oracle
    import workloads as W
    L = oracle.lib()
    spu = samples_per_unit()
    res = {}
    inputs = inputs if inputs is not None else {}

    def timed(name, n_units, make, chunk):
        fn = make(n_units)
        sl = [(lo, min(lo + chunk, n_units)) for lo in range(0, n_units, chunk)]
        t = time.perf_counter()
        oracle.run_parallel(fn, sl, threads)
        res[name] = (n_units, n_units * spu[name], time.perf_counter() - t)

    def params(key, gen):
        if key not in inputs:
            inputs[key] = gen()
        return inputs[key]

    for name in units:
        n = int(units[name])
        if n <= 0:
            continue
        if name in ("cfg2_gaussian", "cfg2_uniform"):
            p2 = params(("cfg2", n), lambda: {k: v.numpy() for k, v in
                                              W.cfg2_params(n, seed=7).items()})
            out = np.empty(n, np.float32)
            f = L.orc_gaussian_f32 if name == "cfg2_gaussian" else L.orc_uniform_f32
            k0, k1 = ("mu", "sigma") if name == "cfg2_gaussian" else ("a", "b")
            timed(name, n, lambda m: (lambda lo, hi: f(
                7, 0, 0, p2[k0][lo:].ctypes.data, p2[k1][lo:].ctypes.data,
                out[lo:].ctypes.data, lo, hi - lo)), 1 << 16)
        elif name == "cfg3_gamma":
            p3 = params(("cfg3", n), lambda: {k: v.numpy() for k, v in
                                              W.cfg3_params(n, seed=11).items()})
            o3 = np.empty(n); t3 = np.empty(n, np.uint8)
            timed(name, n, lambda m: (lambda lo, hi: L.orc_gamma_f64(
                11, 0, 0, p3["alpha"][lo:].ctypes.data, p3["beta"][lo:].ctypes.data,
                o3[lo:].ctypes.data, t3[lo:].ctypes.data, lo, hi - lo)), 1 << 14)
        elif name == "cfg4_dirichlet":
            a4 = params(("cfg4", n), lambda: W.cfg4_params(n, 256, seed=3).numpy())
            o4 = np.empty_like(a4); t4 = np.empty(a4.shape, np.uint8)
            scratch = np.empty((threads, 256))
            slot = {}
            lock = threading.Lock()

            def dirichlet(lo, hi):
                tid = threading.get_ident()
                with lock:
                    j = slot.setdefault(tid, len(slot))
                L.orc_dirichlet_f32(3, 0, 0, a4[lo:].ctypes.data, 256, o4[lo:].ctypes.data,
                                    t4[lo:].ctypes.data, lo, hi - lo, scratch[j].ctypes.data)
            timed(name, n, lambda m: dirichlet, 256)
        elif name == "cfg1_gibbs":
            ox = np.empty((1000, n)); oy = np.empty((1000, n))
            tot = np.zeros((n, 272))

            def gibbs1(lo, hi):
                # one oracle call per chain slice (samples are [sweep][chain]
                # within the slice: the slice's own contiguous output)
                bx = np.empty((1000, hi - lo)); by = np.empty((1000, hi - lo))
                L.orc_gibbs_triangle(42, lo, 0, hi - lo, 1000, None, None, 0, bx.ctypes.data,
                                     by.ctypes.data, None, None, tot[lo].ctypes.data)
            timed(name, n, lambda m: gibbs1, 16)
        elif name == "cfg5_gibbs":
            tot = np.zeros((max(1, n // 64 + 1), 272))
            blk = 64

            def gibbs5(lo, hi):
                # units lo..hi-1 of the subset = chains (u // 64) * stride5 * 64 + u % 64
                for u0 in range(lo, hi, blk):
                    u1 = min(hi, (u0 // blk + 1) * blk)
                    c0 = (u0 // blk) * stride5 * blk + u0 % blk
                    L.orc_gibbs_triangle(42, c0, 0, u1 - u0, 4096, None, None, 0, None, None,
                                         None, None, tot[u0 // blk].ctypes.data)
            timed(name, n, lambda m: gibbs5, blk)
    return res


def _mix_value(res, units_full):
    """Gsamples/s of the FULL step mix from per-config measured rates."""
    spu = samples_per_unit()
    t = sum(units_full[k] * spu[k] / (res[k][1] / res[k][2]) for k in units_full)
    return sum(units_full[k] * spu[k] for k in units_full) / t / 1e9


def cpu_baseline():
    """The oracle as it stands on the GPU box's host cores:
    cfg1-cfg4 at FULL size on all P cores; cfg5 on a stride subset of its
    chains (every 16th block of 64 chains = 1/16, full 4096 sweeps); each
    config again on ONE core on a bounded sample; the CPU model from lscpu."""
    P = _cores()
    fu = full_units()
    inputs = {}
    units_p = dict(fu)
    units_p["cfg5_gibbs"] = fu["cfg5_gibbs"] // 16
    res_p = oracle_run(units_p, P, stride5=16, inputs=inputs)
    inputs.clear()
    units_1 = {"cfg1_gibbs": fu["cfg1_gibbs"] // 8, "cfg2_gaussian": 1 << 22,
               "cfg2_uniform": 1 << 22, "cfg3_gamma": 1 << 21, "cfg4_dirichlet": 8192,
               "cfg5_gibbs": fu["cfg5_gibbs"] // 2048}
    res_1 = oracle_run(units_1, 1, stride5=2048, inputs=inputs)
    rate = lambda r: {k: round(v[1] / v[2] / 1e6, 3) for k, v in r.items()}  # noqa: E731
    return {"value": round(_mix_value(res_p, fu), 6), "unit": UNIT, "cores": P, "kind": "oracle",
            "cpu_model": cpu_model(),
            "value_1core": round(_mix_value(res_1, fu), 6),
            "sample": ("P cores: cfg1-cfg4 at full size (units " +
                       ", ".join(f"{k} {v[0]} in {v[2]:.2f}s" for k, v in res_p.items()) +
                       "); cfg5 every 16th block of 64 chains (1/16 of 2^24, 4096 sweeps). "
                       "1 core: bounded samples (" +
                       ", ".join(f"{k} {v[0]} in {v[2]:.2f}s" for k, v in res_1.items()) +
                       "). value = the full step's samples / the sum of each config's "
                       "full-size time at its measured rate"),
            "per_config_Msamples_per_s": rate(res_p),
            "per_config_Msamples_per_s_1core": rate(res_1)}


def step_samples():
    import workloads as W
    return {"cfg1_gibbs": 2 * W.CFG1["n_chains"] * W.CFG1["n_sweeps"],
            "cfg2_gaussian": W.CFG2["n"], "cfg2_uniform": W.CFG2["n"], "cfg3_gamma": W.CFG3["n"],
            "cfg4_dirichlet": W.CFG4["n_docs"] * W.CFG4["k"],
            "cfg5_gibbs": 2 * W.CFG5["n_chains"] * W.CFG5["n_sweeps"]}


def step_config(world, small=False, scaling="strong"):
    """The `config` object of a bench line (both arms): the workload of one step."""
    where = ("sharded over the N GPUs (strong scaling: fixed totals)" if scaling == "strong"
             else "per GPU (weak scaling: N times the totals)")
    return {"workload": "one step = BASELINE.json configs[0..4] at full size, " + where +
                        " (cfg1 Gibbs 1024x1000 + cfg2 Gaussian&uniform 2^28 f32 + cfg3 "
                        "Gamma 2^26 f64 + cfg4 Dirichlet 1e6x256 f32 + cfg5 Gibbs "
                        "2^24x4096)" + (" [--small: NOT a bench number]" if small else ""),
            "sample_unit": "one output deviate (Gibbs: one conditional draw)",
            "samples_per_gpu_step": sum(step_samples().values()),
            "l2": "inputs larger than L2 (each step streams ~9 GB of parameters/outputs)",
            "dtypes": {"cfg1": "f64", "cfg2": "f32", "cfg3": "f64",
                       "cfg4": "f32 io, f64 internal", "cfg5": "f64"},
            "parallelism": f"dp{world} (disjoint Philox counter ranges; {scaling} scaling)"}


def reference_arm(args):
    """--impl reference: the oracle, as it stands, timed on the host cores.
    Each step is a bounded sample of the same workload -- the same fraction f
    of every config's units (cfg5: a stride subset of its chains), parameters
    by the same recipe -- sized so the W + K steps end in a few minutes;
    ms_per_step is the measured wall time of such a step."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    P = _cores()
    fu = full_units()

    def units_for(f):
        u = {k: max(1, int(round(v * f))) for k, v in fu.items()}
        return u, max(1, int(round(1 / f)))
    budget_total = args.ref_budget_s
    per_step = max(0.5, budget_total / max(1, args.steps + args.warmup))
    f0 = 1.0 / 4096
    u0, st0 = units_for(f0)
    probe = oracle_run(u0, P, stride5=st0)
    t0 = sum(v[2] for v in probe.values())
    f = min(1.0, f0 * per_step / max(t0, 1e-3))
    units, stride = units_for(f)
    inputs = {}
    for _ in range(args.warmup):
        oracle_run(units, P, stride5=stride, inputs=inputs)
    tot_s, tot_samples, last = 0.0, 0, None
    for _ in range(args.steps):
        r = oracle_run(units, P, stride5=stride, inputs=inputs)
        tot_s += sum(v[2] for v in r.values())
        tot_samples += sum(v[1] for v in r.values())
        last = r
    v = tot_samples / tot_s / 1e9
    desc = (f"each step: fraction {f:.3g} of every config's units on {P} cores ("
            + ", ".join(f"{k} {u[0]} units" for k, u in last.items())
            + f"; cfg5 chains at stride {stride} in blocks of 64), parameters by each "
              "config's recipe at that size; value = samples / measured oracle time")
    out = {"metric": METRIC, "value": round(v, 6), "unit": UNIT,
           "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(tot_s / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": step_config(int(os.environ.get("WORLD_SIZE", 1)), scaling=args.scaling),
           "cpu_baseline": {"value": round(v, 6), "unit": UNIT, "cores": P, "kind": "oracle",
                            "cpu_model": cpu_model(), "sample": desc,
                            "per_config_Msamples_per_s":
                                {k: round(x[1] / x[2] / 1e6, 3) for k, x in last.items()}},
           "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="brng", choices=["brng", "reference"])
    ap.add_argument("--small", action="store_true", help="1/64 sizes (functional check only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="e2e steps (default: --steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: total oracle seconds for W + K steps")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the configs' fixed totals sharded over the N GPUs "
                         "(default); weak: every GPU the full configs")
    ap.add_argument("--no-weak", action="store_true",
                    help="strong scaling at N > 1: skip the secondary weak-scaling run")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
