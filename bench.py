#!/usr/bin/env python
"""Benchmark of the batched Hopf-formula evaluator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric: Hopf evaluations per second (phi and grad phi written) at n = 1000 — BASELINE config 3
(J = 1/2(<x,D^-1 x> - 1), H = ||.||_2, M = 1e5 points per GPU, x ~ N(0,I), t ~ U[0,2]).
A "step" is one pass of the whole hot path (stage, (3.4a), (3.4b), (3.4c),
stopping test with masking/refill, phi/grad output) over one batch of M points = one
hopf_eval_diag launch.  Multi-GPU (torchrun): every rank evaluates its own M points (weak
scaling, shards by global index, no data-path collective); the time is the max over ranks.

value      device throughput with X, t resident in HBM (inputs 400 MB > 126 MB L2, no flush needed)
e2e        same metric through hopf_eval_diag_host: pinned host X,t -> device -> host phi,grad,iters
roofline   dominant kernel vs the FP32 ALU peak (148 SMs x 128 lanes x 2 flop x 1965 MHz)
cpu_baseline  the fp64 oracle (oracle/, as it stands) on the host cores, bounded sample
--impl reference  times that oracle as the reference arm (rank 0 only under torchrun)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1605_01799_b200 import inputs, shard  # noqa: E402

METRIC = "Hopf evals/sec (phi+grad phi) at n=1000"
UNIT = "evals/s"
SM_COUNT_NOMINAL = 148
FP32_LANES_PER_SM = 128
# algorithmic FP32 flops per coordinate-iteration: update + the paper's test
# ell (NEXT-2): (3.4a) + u 6, inside test 3, one Newton step on mu 8 (the warm-started steady
# state), d' and b' 5, the test sums 5
# linf (NEXT-2): (3.4a) + u 6, one evaluation of the l1-ball sums 2, d' = clamp 2, b' 1, the
# test sums 5 (min / max / compare-select counted as one flop)
FLOPS_PER_COORD_ITER = {"l2": 17, "l1": 14, "wl1": 14, "ell": 27, "linf": 16}
# NEXT-3 (J = 1/2||.||_1^2 or 1/2||.||_inf^2): z = d - b + x/lambda 2, one evaluation of the
# active-set sums 2, v = clamp / shrink 2, sv 3, u 1, then the H update and the sd, sb sums:
# l1/wl1 4 + 6, l2 3 + 6, linf 2 + 2 + 6
FLOPS_NORMSQ = {"l1": 20, "wl1": 20, "l2": 19, "linf": 20}
# ||.||_A (NEXT-2): the two rotations Q^T u and Q d~ (2 n FMAs each = 4 n flops per coordinate)
# plus the diagonal iteration with one ellipsoid Newton evaluation (27): 4 n + 27
# per-point HBM bytes: x (4n) + grad (4n) + t, phi, iters (12)
CPU_SAMPLE = {"c1": 1024, "c2": 1_000_000, "c3": 100_000, "c4": 4096, "c5": 100_000, "c5d": 2048,
              "c2h": 200_000, "c2e": 200_000,
              "c2i": 200_000, "t5": 1_000_000, "t4a": 200_000}
CPU_SAMPLE_DEFAULT = 200_000   # e.g. the paper-protocol workloads p<n>_<id|diag>_<l1|l2>
CPU_MIN_SECONDS = 10.0
L2_BYTES = 126 * 1024 * 1024


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def clocks_sampler(uuid):
    q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                 "-lms", "100"] + (["-i", uuid] if uuid else []),
                                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except Exception:
        return None


def clocks_summary(proc):
    if proc is None:
        return None
    proc.terminate()
    try:
        out, _ = proc.communicate(timeout=5)
    except Exception:
        proc.kill()
        return None
    sm, smax, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in out.strip().splitlines():
        f = [x.strip() for x in line.split(",")]
        if len(f) < 7:
            continue
        try:
            sm.append(float(f[0]))
            smax.append(float(f[1]))
        except ValueError:
            continue
        for nm, v in zip(names, f[3:7]):
            if v.lower() == "active":
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
            "samples": len(sm)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_traffic(config):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def cpu_baseline_run(wl, sample, min_seconds=0.0):
    """Oracle throughput on the first `sample` points, repeated until min_seconds elapsed."""
    import oracle
    X, t = inputs.points(wl, 0, sample)
    t0 = time.perf_counter()
    reps = 0
    while True:
        _oracle_once(wl, X, t)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return sample * reps / dt, dt, oracle.threads(), reps


def _oracle_once(wl, X, t):
    import oracle
    if wl.kind == "diag":
        oracle.eval_diag(X, t, wl.D, wl.c, wl.gamma, wl.h, wl.w, lam=wl.lam,
                         max_iter=wl.max_iter, tol=wl.tol)
    elif wl.kind == "union":
        oracle.eval_union(X, t, wl.Dk, wl.Ck, wl.gammak, wl.h, lam=wl.lam, max_iter=wl.max_iter,
                          tol=wl.tol)
    elif wl.kind == "maxh":
        kinds, av, Wm = wl.maxh
        oracle.eval_maxh(X, t, wl.D, None, wl.gamma, kinds, av, Wm, lam=wl.lam,
                         max_iter=wl.max_iter, tol=wl.tol)
    elif wl.kind == "distance":
        oracle.distance_union(X, wl.Dk, wl.Ck, wl.gammak, lam=wl.lam, max_iter=wl.max_iter,
                              tol=wl.tol, stol=1e-5)
    elif wl.kind == "ella":
        oracle.eval_diag_A(X, t, wl.D, None, wl.gamma, wl.A, lam=wl.lam, max_iter=wl.max_iter,
                           tol=wl.tol)
    elif wl.kind == "normsq":
        oracle.eval_normsq(X, t, wl.jk, wl.gamma, wl.h, wl.w, lam=wl.lam, max_iter=wl.max_iter,
                           tol=wl.tol)
    else:
        oracle.eval_dense(X, t, wl.Q, wl.Lam, wl.gamma, wl.h, lam=wl.lam, max_iter=wl.max_iter,
                          tol=wl.tol)


def run_reference(args, wl):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    sample = args.cpu_sample or CPU_SAMPLE.get(wl.name, CPU_SAMPLE_DEFAULT)
    for _ in range(args.warmup):
        cpu_baseline_run(wl, max(1, sample // 8))
    times = []
    for _ in range(args.steps):
        v, dt, cores, _ = cpu_baseline_run(wl, sample)
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = sample / (ms / 1e3)
    line = {"metric": metric_name(wl),
            "value": value, "unit": UNIT, "impl": "reference", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE law)",
            "config": config_dict(wl, ws),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"first {sample} points of {wl.name} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def metric_name(wl):
    if wl.kind == "maxh":
        return f"Hopf evals/sec ({wl.name}: H = min of {len(wl.maxh[0])} Hamiltonians, n={wl.n})"
    if wl.kind == "ella":
        return f"Hopf evals/sec ({wl.name}: J = 1/2<x, D^-1 x>, H = ||.||_A full SPD, n={wl.n})"
    if wl.kind == "normsq":
        jn = "1/2||.||_1^2" if wl.jk == "l1sq" else "1/2||.||_inf^2"
        return f"Hopf evals/sec ({wl.name}: J = {jn}, H = {wl.h}, n={wl.n})"
    if wl.kind == "distance":
        return f"closest-point queries/sec ({wl.name}: union of K={wl.Dk.shape[0]} ellipsoids, n={wl.n})"
    return METRIC if wl.name == "c3" else f"Hopf evals/sec ({wl.name}, n={wl.n})"


def config_dict(wl, ws, flush=False):
    d = {"workload": f"{wl.name}: n={wl.n}, M={wl.M} points per GPU, H={wl.h}, J={wl.kind}",
         "n": wl.n, "M_per_gpu": wl.M, "global_points": wl.M * ws, "lambda": wl.lam,
         "tol": wl.tol, "max_iter": wl.max_iter, "parallelism": f"dp{ws} (point shards)",
         "l2_flush": ("256 MB write before every step (working set below 2 x the 126 MB L2); "
                      "steps timed one by one, flush outside the event pairs") if flush else
                     "none needed: per-step inputs+outputs exceed twice the 126 MB L2"}
    if wl.kind in ("union", "distance"):
        d["K"] = int(wl.Dk.shape[0])
    if wl.kind == "distance":
        d["workload"] = (f"{wl.name}: distance/projection to the union of K={d['K']} ellipsoids, "
                         f"n={wl.n}, M={wl.M} query points per GPU (Newton in s, P:1085-1108)")
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--M", type=int, default=None, help="points per GPU (default: the config's)")
    ap.add_argument("--n", type=int, default=None, help="dimension override (experiments; default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    wl = inputs.config(args.config, M=args.M, n=args.n)
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist
    import paper_1605_01799_b200 as hb

    ws, rank, local = dist_env()
    if os.environ.get("HOPF_BENCH_BACKEND", "nccl") != "nccl":
        local = local % torch.cuda.device_count()   # the gloo test: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        # HOPF_BENCH_BACKEND=gloo: a test of the multi-rank code paths with several ranks on one GPU
        # (NCCL refuses two ranks on one device); the timed numbers of such a run mean nothing
        backend = os.environ.get("HOPF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    L = hb.lib()

    # ---- inputs: this rank's shard of the global points (generated by global index) ----------
    M = wl.M
    r0, r1 = shard.weak_range(M, rank)
    wl_g = inputs.config(args.config, M=M * ws, n=args.n)
    Xh, th = inputs.points(wl_g, r0, r1)
    X = torch.from_numpy(Xh).to(dev)
    t = torch.from_numpy(th).to(dev)
    n = wl.n
    f32 = lambda a: None if a is None else torch.as_tensor(a, dtype=torch.float32, device=dev)
    phi = torch.empty(M, device=dev)
    grad = torch.empty((M, n), device=dev)
    iters = torch.empty(M, dtype=torch.int32, device=dev)
    out = (phi, grad, iters)
    stream = torch.cuda.current_stream(dev)

    if wl.kind == "diag":
        D, c, w = f32(wl.D), f32(wl.c), f32(wl.w)
        step = lambda: hb.eval_diag(X, t, D, c, wl.gamma, wl.h, w, wl.lam, wl.max_iter, wl.tol,
                                    out=out, stream=stream)
    elif wl.kind == "union":
        Dk, Ck, gk = f32(wl.Dk), f32(wl.Ck), f32(wl.gammak)
        Y = torch.empty((M, n), device=dev)
        kst = torch.empty(M, dtype=torch.int32, device=dev)

        def step():
            rc = L.hopf_eval_union(M, n, wl.K, X.data_ptr(), t.data_ptr(), Dk.data_ptr(),
                                   Ck.data_ptr(), gk.data_ptr(), hb.H_KINDS[wl.h], None,
                                   float(wl.lam), wl.max_iter, float(wl.tol), phi.data_ptr(),
                                   grad.data_ptr(), iters.data_ptr(), Y.data_ptr(),
                                   kst.data_ptr(), None, stream.cuda_stream)
            hb._check(rc, "hopf_eval_union")
    elif wl.kind == "maxh":
        kinds, av, Wm = wl.maxh
        D, Wd = f32(wl.D), f32(Wm)
        mres = {}

        def step():
            mres["r"] = hb.eval_maxh(X, t, D, None, wl.gamma, kinds, av, Wd, wl.lam, wl.max_iter,
                                     wl.tol, out=out, stream=stream)
    elif wl.kind == "ella":
        import numpy as _np
        lam_A, Q_A = _np.linalg.eigh(wl.A)
        D, Qd, Ld = f32(wl.D), f32(_np.ascontiguousarray(Q_A)), f32(lam_A)
        step = lambda: hb.eval_diag_A(X, t, D, None, wl.gamma, Qd, Ld, wl.lam, wl.max_iter, wl.tol,
                                      out=out, stream=stream)
    elif wl.kind == "normsq":
        w = f32(wl.w)
        step = lambda: hb.eval_normsq(X, t, wl.jk, wl.gamma, wl.h, w, wl.lam, wl.max_iter, wl.tol,
                                      out=out, stream=stream)
    elif wl.kind == "distance":
        Dk, Ck, gk = f32(wl.Dk), f32(wl.Ck), f32(wl.gammak)
        dres = {}

        def step():
            dres["r"] = hb.distance_union(X, Dk, Ck, gk, wl.lam, wl.max_iter, wl.tol,
                                          stream=stream)
    else:
        plan = hb.DensePlan(wl.Q, wl.Lam, wl.lam)
        step = lambda: hb.eval_dense(X, t, plan, wl.gamma, wl.h, None, wl.max_iter, wl.tol,
                                     out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    iters_np = iters.cpu().numpy() if wl.kind != "distance" else dres["r"][5].cpu().numpy()
    launches_per_step = hb.last_launch_count()
    kernel_name = hb.last_kernel()
    # total split Bregman iterations of one step (all solves: union sets, Newton evaluations),
    # from the library's instrumentation counter in one extra untimed step
    inner_iters = None
    if wl.kind in ("diag", "union", "distance", "maxh", "normsq", "ella"):
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        hb.set_iteration_counter(cnt)
        step()
        torch.cuda.synchronize(dev)
        hb.set_iteration_counter(None)
        inner_iters = int(cnt.item())
    import ctypes
    _th, _bl = ctypes.c_int32(0), ctypes.c_int32(0)
    L.hopf_last_launch_config(ctypes.byref(_th), ctypes.byref(_bl))
    launch_cfg = {"threads_per_block": _th.value, "blocks": _bl.value}

    uuid = None
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        pass
    smi = clocks_sampler(uuid)
    time.sleep(0.3)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # per-step working set (inputs + outputs); below twice the 126 MB L2 every step is preceded
    # by an L2 flush (a 256 MB write, outside its own event pair) and the steps are timed one by one
    per_point = 8 * n + 12 + (4 * n + 4 if wl.kind in ("union", "distance") else 0)
    flush = M * per_point < 2 * L2_BYTES
    if flush:
        scrub = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            scrub.fill_(1.0)
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize(dev)
        ms_total = sum(a.elapsed_time(b) for a, b in evs)
    else:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        ms_total = ev0.elapsed_time(ev1)
    if ws > 1:
        dist.barrier()
    clocks = clocks_summary(smi)
    if ws > 1:
        tm = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms_total = float(tm.item())
    ms_step = ms_total / args.steps
    value = M * ws / (ms_step / 1e3)

    # ---- result gather over NCCL (N > 1): the method's only collective -------------
    gather = None
    if ws > 1:
        def timed(fn, reps=3):
            fn()
            torch.cuda.synchronize(dev)
            dist.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(reps):
                fn()
            g1.record(stream)
            torch.cuda.synchronize(dev)
            tm = torch.tensor([g0.elapsed_time(g1) / reps], device=dev, dtype=torch.float64)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            return float(tm.item())
        ms_small = timed(lambda: shard.gather_results([phi, iters]))
        ms_grad = timed(lambda: shard.gather_results([grad]))
        gbytes = grad.numel() * 4 * ws
        gather = {"what": "all_gather_into_tensor of every rank's results (NCCL), outside the timed step",
                  "phi_iters_ms": ms_small, "grad_ms": ms_grad,
                  "grad_bytes_gathered": gbytes,
                  "grad_GBps_per_rank_in": gbytes * (ws - 1) / ws / (ms_grad / 1e3) / 1e9}
        if wl.kind == "diag":
            # the evaluation chunk by chunk with each chunk's phi, grad, iters all-gathered on NCCL's
            # stream while the next chunk computes: end-to-end step with the gather
            full = (torch.empty(M * ws, device=dev), torch.empty((M * ws, n), device=dev),
                    torch.empty(M * ws, dtype=torch.int32, device=dev))
            Dg, cg, wg = f32(wl.D), f32(wl.c), f32(wl.w)

            def ev_chunk(lo, hi):
                o = (phi[lo:hi], grad[lo:hi], iters[lo:hi])
                hb.eval_diag(X[lo:hi], t[lo:hi], Dg, cg, wl.gamma, wl.h, wg, wl.lam, wl.max_iter,
                             wl.tol, out=o, stream=stream)
                return o
            chunk = max(1, M // 8)
            ms_pipe = timed(lambda: shard.eval_gather_pipelined(ev_chunk, M, chunk, full))
            gather.update({"pipelined_step_ms": ms_pipe, "pipelined_chunks": -(-M // chunk),
                           "compute_only_step_ms": ms_step,
                           "pipelined_value": M * ws / (ms_pipe / 1e3),
                           "pipelined_what": "eval + all_gather of phi, grad, iters per chunk, "
                                             "gather of chunk i overlapped with compute of chunk i+1"})

    # ---- end to end through the host-buffer entry point (diag path) ----------------------------
    e2e = None
    if not args.no_e2e and wl.kind == "diag":
        Xp = torch.from_numpy(Xh).pin_memory()
        tp = torch.from_numpy(th).pin_memory()
        outh = (torch.empty(M, pin_memory=True), torch.empty((M, n), pin_memory=True),
                torch.empty(M, dtype=torch.int32, pin_memory=True))
        Dd, cd, wd = f32(wl.D), f32(wl.c), f32(wl.w)
        e2e_step = lambda: hb.eval_diag_host(Xp, tp, Dd, cd, wl.gamma, wl.h, wd, wl.lam,
                                             wl.max_iter, wl.tol, out=outh)
        for _ in range(2):
            e2e_step()
        if ws > 1:
            dist.barrier()
        ksteps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(ksteps):
            e2e_step()
        el = time.perf_counter() - t0   # the call is synchronous: results are in host memory
        if ws > 1:
            tm = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            el = float(tm.item())
        e2e = {"value": M * ws * ksteps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(Xp.numel() * 4 + tp.numel() * 4),
               "d2h_bytes_per_step": int(M * 4 + M * n * 4 + M * 4),
               "api": "hopf_eval_diag_host (pinned host buffers, chunked H2D/kernel/D2H pipeline)"}
    elif not args.no_e2e:
        # no host-buffer entry point for these kinds: pinned H2D of x and t, the call, D2H of every
        # result the call writes (phi, grad, iters; union: + y, k*; maxh: + winner; distance: its six)
        Xp = torch.from_numpy(Xh).pin_memory()
        tp = torch.from_numpy(th).pin_memory()

        def results():
            if wl.kind == "union":
                return [phi, grad, iters, Y, kst]
            if wl.kind == "maxh":
                return list(mres["r"])
            if wl.kind == "distance":
                return list(dres["r"])
            return list(out)
        outh = [torch.empty(r.shape, dtype=r.dtype, pin_memory=True) for r in results()]

        def e2e_step():
            X.copy_(Xp, non_blocking=True)
            t.copy_(tp, non_blocking=True)
            step()
            for hbuf, dbuf in zip(outh, results()):
                hbuf.copy_(dbuf, non_blocking=True)
            torch.cuda.synchronize(dev)
        for _ in range(2):
            e2e_step()
        if ws > 1:
            dist.barrier()
        ksteps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(ksteps):
            e2e_step()
        el = time.perf_counter() - t0
        if ws > 1:
            tm = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            el = float(tm.item())
        api = {"normsq": "hopf_eval_normsq", "ella": "hopf_eval_diag_A", "union": "hopf_eval_union",
               "maxh": "hopf_eval_maxh", "distance": "hopf_distance_union",
               "dense": "hopf_eval_dense"}.get(wl.kind, wl.kind)
        e2e = {"value": M * ws * ksteps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(Xp.numel() * 4 + tp.numel() * 4),
               "d2h_bytes_per_step": int(sum(h.numel() * h.element_size() for h in outh)),
               "api": f"{api} with torch pinned copies on the same stream"}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ---------------------------------------------------
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    conv = iters_np[iters_np > 0]
    roof = None
    if wl.kind in ("diag", "union", "distance", "maxh", "normsq", "ella"):
        it_sum = float(inner_iters)
        # algorithmic HBM bytes per point: diag x in, grad out (4n each) + t, phi, iters;
        # union / distance also write y (closest point / projection) and k*
        hbm_per_point = (8 * n + 12) if wl.kind in ("diag", "maxh", "normsq", "ella") else (12 * n + 16)
        fpc = (FLOPS_NORMSQ[wl.h] if wl.kind == "normsq" else (4 * n + 27 if wl.kind == "ella"
               else FLOPS_PER_COORD_ITER["l1" if wl.kind == "maxh" else wl.h]))
        flops = it_sum * n * fpc
        achieved = flops / (ms_step / 1e3) / 1e12
        peak = sms * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
        roof = {"kernel": kernel_name, "bound": "alu", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": load_traffic(wl.name),
                "peak_basis": f"{sms} SMs x 128 FP32 lanes x 2 flop x {sm_max:.0f} MHz (guide unit "
                              "counts, max SM clock)",
                "algorithmic_flops_per_launch": flops,
                "inner_iterations_per_launch": inner_iters,
                "flops_per_coord_iter": fpc,
                "mean_iters": float(conv.mean()) if conv.size else None,
                "hbm_bytes_per_launch": M * hbm_per_point,
                "hbm_GBps": M * hbm_per_point / (ms_step / 1e3) / 1e9}
        if clocks:
            roof["frac_at_measured_clock"] = achieved / (sms * FP32_LANES_PER_SM * 2 *
                                                         clocks["sm_mhz"] * 1e6 / 1e12)
        # below the ridge (few iterations per point, e.g. J = 1/2||.||^2: 3 iterations) the
        # launch is bound by its HBM traffic: report it against the measured copy bandwidth
        hbm_peak = float(peaks.get("hbm_gbs", 6530.6))
        if flops / (M * hbm_per_point) < peak * 1e3 / hbm_peak:
            roof.update({"bound": "hbm", "achieved": roof["hbm_GBps"], "peak": hbm_peak,
                         "unit": "GB/s", "frac": roof["hbm_GBps"] / hbm_peak,
                         "peak_basis": "measured HBM copy bandwidth (MEASURED_PEAKS.json)",
                         "alu_frac": achieved / peak})
    else:
        # dense: the v-update GEMM dominates: algorithmic 2 n^2 flops per point-iteration; the
        # tensor-core kernel executes 3 fp16 products (hi/lo split) per algorithmic one
        it_sum = float(np.abs(iters_np[iters_np != inputs_invalid()]).sum())
        flops = it_sum * 2.0 * n * n
        achieved = flops / (ms_step / 1e3) / 1e12
        tc = (n == 256 and wl.h != "l2")
        bf16 = float(peaks.get("bf16_tflops", 1645.3))
        peak = bf16 if tc else sms * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
        roof = {"kernel": kernel_name, "bound": "tensor" if tc else "alu", "achieved": achieved,
                "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": load_traffic(wl.name),
                "peak_basis": ("measured dense bf16 cuBLAS burst (MEASURED_PEAKS.json); fp16 "
                               "kind::f16 runs at the bf16 rate") if tc else "FP32 SIMT peak",
                "algorithmic_flops_per_launch": flops,
                "executed_tensor_flops_per_launch": 3 * flops if tc else None,
                "executed_frac": 3 * achieved / peak if tc else None,
                # the target's own metric, from the committed ncu capture of this build
                "tensor_pipe_active_frac_ncu": (load_traffic("_tensor_pipe_active_pct") or {}).get(wl.name, 0) / 100
                if tc else None,
                "mean_iters": float(conv.mean()) if conv.size else None}
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        sample = min(args.cpu_sample or CPU_SAMPLE.get(wl.name, CPU_SAMPLE_DEFAULT), wl.M)
        v, dt, cores, reps = cpu_baseline_run(wl, sample, CPU_MIN_SECONDS)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first {sample} points of {wl.name} x {reps} passes "
                         f"({dt:.1f} s of the fp64 oracle, OpenMP over points)"}

    line = {"metric": metric_name(wl),
            "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; BASELINE config law)", "config": config_dict(wl, ws, flush),
            "clocks": clocks, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gather": gather,
            "gpu_launches": launches_per_step * args.steps,
            "launch": launch_cfg if wl.kind != "dense" else None,
            "iters": {"min": int(conv.min()) if conv.size else None,
                      "mean": float(conv.mean()) if conv.size else None,
                      "max": int(conv.max()) if conv.size else None,
                      "nonconverged": int(np.sum((iters_np < 0) & (iters_np != inputs_invalid())))}}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def inputs_invalid():
    return -(2 ** 31)


if __name__ == "__main__":
    sys.exit(main())
