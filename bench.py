#!/usr/bin/env python
"""FS-1 hot-path benchmark (driver contract: one JSON line on rank 0).

A "step" is one full FS-1 solve (Algorithm 1: every iteration, the marginal
error at exit and the fused return-line cost) over one batch of synthetic
histogram pairs of BASELINE.json's configuration.  Default workload: configs[2]
("c3": one pair, N = 2^24, fp64 log domain, eps = 1e-4, 1000 iterations) —
BASELINE.json quotes its metric on no particular config, so the bench line is
the largest single-GPU configuration (the HBM-streaming kernel K2, the one the
metric's "achieved HBM GB/s" half is about).  Every other config runs with
--config cK.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl fs1|reference]

Multi-GPU (torchrun, one process per GPU): weak scaling — every rank solves its
own batch of distinct pairs (pair ids rank*B + i, same recipe); the per-pair
results {cost, iters, err, flags} are all-gathered with NCCL inside each step.
"""
from __future__ import annotations

import argparse
import dataclasses
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

import fs1_inputs as gi  # noqa: E402

METRIC = "grid-point Sinkhorn updates/sec (N*iters*batch/s) and achieved HBM GB/s"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(gi.CONFIGS))
    ap.add_argument("--impl", default="fs1", choices=["fs1", "reference"])
    ap.add_argument("--batch", type=int, default=None, help="pairs per GPU (default: config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel", type=int, default=0, help="test-only plan override (0 = automatic choice)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def per_gpu_batch(cfg, args):
    if args.batch:
        return args.batch
    if cfg.name == "c5":
        return 8192          # 65536 pairs over 8 GPUs (BASELINE configs[4])
    return cfg.batch


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- roofline
NOMINAL_HBM_GBS = 8000.0    # the north_star's "~8 TB/s" denominator
MUFU_PER_SM_CLK = 16        # fp32 MUFU ops per SM per clock (tools/ubench.cu, profiles/r02_ubench.txt)
DFMA_PER_SM_CLK = 64        # fp64 FMA per SM per clock (same micro-benchmark)
# fp64 persistent kernels, per update: 2 half-steps x (2 recursion FMAs + 1 combine +
# 5 for the quotient y = tgt / Kx: MUFU.RCP64H seed, 2 Newton FMA pairs, 1 multiply)
DFMA_PER_UPDATE = 16


def launches_per_solve(info, batch):
    """Library kernels one fs1_solve launches: K1, K4, K5 one launch for the whole batch;
    K2 and K3w / K3 one cooperative launch per problem (each preceded by a
    cudaMemsetAsync of its grid-barrier counter, which is not a kernel)."""
    return 1 if info["kernel"].startswith(("persist", "stab", "sep2d64", "sep3d64")) else batch


def roofline(cfg, info, updates, it_run, batch, kern_s, peaks, src, props):
    """Roofline object of the dominant kernel + achieved algorithmic HBM GB/s.

    Algorithmic HBM bytes: a streaming kernel (K2, K3w / K3) reads
    x and the target and writes y once per half-step, 6 words per update (fixed-iteration
    runs: no check word); a persistent kernel (K1) keeps the state on chip and moves 4
    words per grid point per solve (reads a, b; writes u, v)."""
    kern = info["kernel"]
    wb = 8 if cfg.dtype == "f64" else 4
    sms = props.multi_processor_count
    clk = peaks.get("sm_max_mhz", 1965.0)
    onchip = kern.startswith(("persist", "stab", "sep2d64", "sep3d64"))   # one CTA per problem (K1, K4, K5)
    if onchip:
        alg = 4 * wb * cfg.size * batch
    else:
        alg = 6 * wb * updates
    hbm = alg / kern_s / 1e9
    ups = updates / kern_s
    if not onchip:
        peak = peaks.get("hbm_gbs", 6650.0)
        r = {"bound": "hbm", "achieved": hbm, "peak": peak, "unit": "GB/s", "frac": hbm / peak,
             "traffic": profile_traffic(cfg.name), "kernel_ms": kern_s * 1e3,
             "algorithmic_bytes_per_launch": alg / launches_per_solve(info, batch),
             "bytes_per_update": 6 * wb,
             "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
             "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": hbm / NOMINAL_HBM_GBS}
        if kern.startswith("sep2dw"):
            r["note"] = ("the 64 MiB working set stays in L2 (traffic << algorithmic bytes); "
                         "the kernel is MUFU/latency-bound, DESIGN.md §6.4")
        return r, hbm
    ctas = info.get("ctas_per_problem", 1) * batch
    if ctas < sms:
        # fewer CTAs than SMs (C1: one pair on one SM): a latency-bound sequential chain
        return {"bound": "latency", "achieved": kern_s * 1e6 / max(it_run, 1), "peak": None,
                "unit": "us/iteration", "frac": None, "traffic": profile_traffic(cfg.name),
                "kernel_ms": kern_s * 1e3,
                "note": f"{ctas} CTA(s) on {sms} SMs: time per iteration is the figure of merit"}, hbm
    if cfg.dtype == "f64":
        peak = sms * clk * 1e6 * DFMA_PER_SM_CLK / DFMA_PER_UPDATE
        how = f"{sms} SMs x {clk:.0f} MHz x {DFMA_PER_SM_CLK} DFMA/clk / {DFMA_PER_UPDATE} DFMA per update"
    else:
        peak = sms * clk * 1e6 * MUFU_PER_SM_CLK / 2.0
        how = f"{sms} SMs x {clk:.0f} MHz x {MUFU_PER_SM_CLK} MUFU/clk / 2 rcp per update"
    r = {"bound": "alu", "achieved": ups / 1e9, "peak": peak / 1e9, "unit": "Gupdate/s",
         "frac": ups / peak, "traffic": profile_traffic(cfg.name), "kernel_ms": kern_s * 1e3,
         "peak_source": "derived: " + how}
    if kern == "persist_f32_log_E32_W1":
        # context: the instruction-issue bound of this kernel's measured
        # mix (thread-instructions per update from ncu at C2)
        ib = sms * clk * 1e6 * 128 / 25.5
        r["issue_bound"] = ib / 1e9
        r["frac_of_issue_bound"] = ups / ib
    return r, hbm


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def profile_traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(cfg_name)
    return None


# ----------------------------------------------------------------------------- oracle legs
def oracle_sample(cfg, pairs, iters, n=None):
    """Time the oracle (as it stands) on a bounded sample; returns (updates, seconds).
    ``n`` shrinks the grid (same recipe): the large single problems' samples and the
    untimed warm-up calls."""
    from oracle import sinkhorn
    if n is not None:
        cfg = dataclasses.replace(cfg, n=n, m=(n if cfg.ndim == 2 else 1))
    A, B = gi.batch(cfg, pairs)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    t0 = time.perf_counter()
    if cfg.domain == "stabilized":
        from oracle import stabilized
        for p in range(len(pairs)):
            stabilized.solve_stab(A64[p], B64[p], n=cfg.n, h=cfg.h1, eps=cfg.eps, itr_max=iters)
    elif cfg.domain == "scaling" or (cfg.ndim == 1 and cfg.n <= 8192):
        sinkhorn.solve(A64, B64, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=iters,
                       domain="scaling", input_is_log=cfg.input_is_log)
    else:
        sinkhorn.solve(A64, B64, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=iters,
                       domain="log", input_is_log=cfg.input_is_log, apply="recur")
    t = time.perf_counter() - t0
    return cfg.size * iters * len(pairs), t


def oracle_cores():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def sample_plan(cfg):
    """Bounded oracle sample (seconds of CPU work) for the config: (pairs, iterations,
    grid size or None for the config's, description).  The large single problems run the
    same recipe on a shorter grid (the oracle's cost per update does not depend on N)."""
    if cfg.name == "c2":
        return list(range(256)), cfg.itr_max, None, "256 of 4096 pairs, all 500 iterations, dense fp64 (BLAS)"
    if cfg.name == "c5":
        return list(range(8)), 200, None, "8 pairs, 200 of 1000 iterations, dense fp64 (BLAS)"
    if cfg.name == "c1":
        return [0], 700, None, "1 pair, 700 iterations, dense fp64"
    if cfg.name == "c3":
        return [0], 1, 1 << 21, ("1 pair of C3's recipe on 2^21 of its 2^24 points, 1 of 1000 iterations + exit "
                                 "check + cost, plain-C LSE recursion (x87)")
    if cfg.name == "c4":
        return [0], 2, 512, "1 pair of C4's recipe on 512^2 of its 2048^2 points, 2 of 300 iterations, plain-C LSE"
    if cfg.name.startswith("e2s_"):
        it = {500: 2000, 2000: 1000, 8000: 300}.get(cfg.n, 100)
        return [0], it, None, (f"1 of 100 pairs, {it} of {cfg.itr_max} iterations, the stabilised oracle "
                               "(plain C recursions)")
    if cfg.name.startswith(("e1_", "e2_")):
        it = {500: 500, 2000: 50, 8000: 20}.get(cfg.n, 20)
        return [0], it, None, f"1 of 100 pairs, {it} of {cfg.itr_max} iterations, dense fp64"
    if cfg.name.startswith("e3_"):
        it = {10: 1000, 20: 1000, 40: 300, 80: 100, 160: 30}.get(cfg.n, 30)
        return [0], it, None, f"1 of 100 trials, {it} of {cfg.itr_max} iterations, dense fp64 per axis"
    return [0], 1, None, "1 pair, 1 iteration, plain-C LSE recursion"


def host_threads():
    """Rank 0 runs the oracle alone (the other ranks exit): give its BLAS every host core,
    also under torchrun, which sets OMP_NUM_THREADS=1 per process."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=os.cpu_count())
    except Exception:
        return None


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    _limits = host_threads()  # noqa: F841 (kept alive for the run)
    pairs, iters, sn, what = sample_plan(cfg)
    # warm-up steps: the same oracle on a short prefix of the workload (builds the C
    # oracle, starts the BLAS / OpenMP threads); the large configs' full sample would
    # cost seconds per untimed step
    for _ in range(max(1, args.warmup)):
        oracle_sample(cfg, pairs[:1], 1, n=None if cfg.size <= 65536 else 256)
    times = []
    ups = 0
    for _ in range(args.steps):
        u, t = oracle_sample(cfg, pairs, iters, n=sn)
        ups, times = u, times + [t]
    T = sum(times)
    value = ups * len(times) / T
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (fs1_inputs recipe of BASELINE configs)",
            "config": {"workload": cfg.name, "description": cfg.description, "sample": what},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle",
                             "sample": what},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def run_fs1(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2202_10042_b200 import dist as fdist
    from paper_2202_10042_b200 import fs1

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    B = per_gpu_batch(cfg, args)
    total = B * ws                      # weak scaling: B pairs per GPU
    pair_ids = fdist.shard(total, rank, ws)
    A, Bm = gi.batch(cfg, pair_ids)
    tdt = torch.float32 if cfg.dtype == "f32" else torch.float64
    a = torch.from_numpy(A).to(dev)
    b = torch.from_numpy(Bm).to(dev)
    shape = (cfg.n, cfg.m) if cfg.ndim == 2 else None
    spec = fs1.Spec(ndim=cfg.ndim, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, batch=B,
                    dtype=tdt, domain=cfg.domain, input_is_log=cfg.input_is_log,
                    itr_max=cfg.itr_max, tol=cfg.tol, kernel=args.kernel)
    plan = fs1.plan(spec, local)
    u, v = torch.empty_like(a), torch.empty_like(b)
    iters = torch.empty(B, dtype=torch.int32, device=dev)
    err = torch.empty(B, dtype=torch.float64, device=dev)
    flags = torch.empty(B, dtype=torch.int32, device=dev)
    cost = torch.empty(B, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.solve_into(a, b, u, v, iters, err, flags, cost)
        if ws > 1:   # the one collective of the path: gather per-pair results (NCCL)
            fdist.gather_results(fdist.pack_results(cost, err, iters, flags), total)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        for i in range(args.steps):
            flush.zero_()                              # L2 flush between timed steps (untimed)
            ev[i][0].record(stream)
            kev[i][0].record(stream)
            plan.solve_into(a, b, u, v, iters, err, flags, cost)
            kev[i][1].record(stream)
            if ws > 1:
                fdist.gather_results(fdist.pack_results(cost, err, iters, flags), total)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    kern_ms = [s.elapsed_time(e) for s, e in kev]
    T = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(T, op=dist.ReduceOp.MAX)
    total_s = T.item() / 1e3
    it_run = int(iters.max().item())
    # updates this rank did per step: N x (executed iterations) summed over its pairs
    updates_per_step_rank = cfg.size * int(iters.to(torch.int64).sum().item())
    U = torch.tensor([updates_per_step_rank], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(U, op=dist.ReduceOp.SUM)
    updates_per_step = U.item()
    value = updates_per_step * args.steps / total_s
    kern_avg_s = statistics.mean(kern_ms) / 1e3

    # ---- end-to-end through the public API with host buffers (pinned): every step copies
    # its inputs host -> device, solves, and reads its costs back.  Steps are pipelined the
    # way a serving loop runs them: step k+1's inputs are copied on a second stream while
    # step k solves (double-buffered device inputs, event-ordered reuse).
    e2e = None
    if not args.no_e2e:
        ha = torch.from_numpy(A).pin_memory()
        hb = torch.from_numpy(Bm).pin_memory()
        hcs = [torch.empty(B, dtype=torch.float64).pin_memory() for _ in range(2)]
        da = [torch.empty_like(a) for _ in range(2)]
        db = [torch.empty_like(b) for _ in range(2)]
        cs = torch.cuda.Stream(dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        kw = dict(h=cfg.h1, eps=cfg.eps, itr_max=cfg.itr_max, tol=cfg.tol, domain=cfg.domain,
                  input_is_log=cfg.input_is_log, shape=shape, h2=cfg.h2 if cfg.ndim == 2 else None,
                  kernel=args.kernel)

        def issue_copy(k):
            with torch.cuda.stream(cs):
                if k >= 2:
                    cs.wait_event(freed[k % 2])
                da[k % 2].copy_(ha, non_blocking=True)
                db[k % 2].copy_(hb, non_blocking=True)
                ready[k % 2].record(cs)

        def run_steps(nsteps):
            issue_copy(0)
            for k in range(nsteps):
                if k + 1 < nsteps:
                    issue_copy(k + 1)
                stream.wait_event(ready[k % 2])
                out = fs1.solve(da[k % 2], db[k % 2], **kw)
                freed[k % 2].record(stream)
                hcs[k % 2].copy_(out["cost"], non_blocking=True)

        run_steps(2)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        run_steps(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        Te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(Te, op=dist.ReduceOp.MAX)
        e2e = {"value": updates_per_step * args.steps / (Te.item() / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(ha.numel() * ha.element_size() + hb.numel() * hb.element_size()),
               "d2h_bytes_per_step": int(hcs[0].numel() * hcs[0].element_size()),
               "pipelined": "inputs of step k+1 copied on a second stream while step k solves"}

    if rank == 0:
        peaks, src = load_peaks()
        props = torch.cuda.get_device_properties(dev)
        clocks = clk.summary()
        info = plan.info()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": sum(step_ms) / len(step_ms),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": cfg.dtype, "data": "synthetic (fs1_inputs recipe of BASELINE configs)",
                "config": {"workload": cfg.name, "description": cfg.description, "pairs_per_gpu": B,
                           "n": cfg.n, "m": cfg.m, "iters": it_run, "domain": cfg.domain,
                           "kernel": info["kernel"], "parallelism": f"batch-sharded x{ws} (weak)",
                           "l2": "flushed between timed steps (256 MiB write, untimed)"},
                "gpu_launches": args.steps * launches_per_solve(info, B),
                "clocks": clocks}
        if cfg.name in gi.PAPER_TABLE1_SECONDS:
            # the paper's own FS-1 number for this exact workload (Table 1, PAPER.md:371-373:
            # seconds per 1000-iteration trial on a 14-core Xeon Gold 5117, CPU): context
            paper_ups = cfg.n * cfg.itr_max / gi.PAPER_TABLE1_SECONDS[cfg.name]
            line["vs_baseline"] = value / paper_ups
            table = "Table 1" if cfg.name.startswith("e1") else "Table 2"
            line["baseline"] = {"value": paper_ups, "unit": UNIT, "source": f"PAPER.md {table} (CPU, "
                                "Xeon Gold 5117), N x iterations / seconds per trial", "hardware": "CPU"}
        line["roofline"], line["hbm_gbs"] = roofline(cfg, info, updates_per_step_rank, it_run, B,
                                                     kern_avg_s, peaks, src, props)
        line["e2e"] = e2e
        if not args.no_cpu_baseline:
            pairs, it, sn, what = sample_plan(cfg)
            oracle_sample(cfg, pairs[:1], 1, n=None if cfg.size <= 65536 else 256)   # warm-up
            u_, t_ = oracle_sample(cfg, pairs, it, n=sn)
            line["cpu_baseline"] = {"value": u_ / t_, "unit": UNIT, "cores": oracle_cores(),
                                    "kind": "oracle", "sample": what, "seconds": t_}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = gi.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_fs1(args, cfg)


if __name__ == "__main__":
    main()
