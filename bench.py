"""Benchmark of the tensor-based sketch hot path (arXiv 2209.14637) on B200.

One step = one pass of the whole hot path over the configured stream:
  local mode-1 Gram of this rank's training shard (3xTF32 tcgen05)  ->  NCCL all-reduce of G (N > 1)
  ->  top-k eigenvectors (sketch S)  ->  batched SCW + per-matrix error on this rank's test shard.
Metric (BASELINE.json): training matrices/s for sketch construction = D_train / step time (the
step includes the test-stream SCW, so this is conservative); strong scaling (D_train fixed).

  python bench.py [--gpus N --steps K --warmup W --config C4]        (torchrun for N > 1)
  python bench.py --impl reference ...                                 (the float64 CPU oracle)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "training matrices/s for sketch construction"
UNIT = "matrices/s"
NOMINAL_TF32_OVER_BF16 = 1.1 / 2.25   # B200_PROFILING.md nominal dense ratio (tf32 1.1 PF, bf16 2.25 PF)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload_desc(c, n_gpus):
    idx = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}.get(c.name, "?")
    kind = "frame-like synthetic stream" if c.offset is not None else "low-rank-plus-noise synthetic stream"
    return {"workload": f"{c.name}: m={c.m} n={c.n} D_train={c.D_train} D_test={c.D_test} k={c.k} r={c.r} "
                        f"(BASELINE.json configs[{idx}], {kind})",
            "m": c.m, "n": c.n, "D_train": c.D_train, "D_test": c.D_test, "k": c.k, "r": c.r,
            "parallelism": f"dp{n_gpus} over the stream index d (one NCCL all-reduce of G)",
            "l2_policy": f"inputs larger than L2 ({c.train_bytes / 1e9:.1f} GB training stream per step)"}


class NvmlClockSampler:
    """SM clocks and throttle reasons sampled every 5 ms through NVML (nvidia_ml_py) in a background
    thread during the timed region; ClockSampler (nvidia-smi -lms) is the fallback."""

    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        import threading
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.rows = []
        self.stop_flag = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_flag.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM), get_reasons(self.h)))
            except Exception:
                pass
            time.sleep(0.005)

    def stop(self):
        self.stop_flag.set()
        self.t.join()
        sm = [r[0] for r in self.rows]
        reasons = sorted({nm for _, bits in self.rows for nm, b in self.REASONS.items() if bits & b})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


def clock_sampler(index):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def dist_setup(n_gpus):
    if n_gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        rank = int(os.environ["RANK"])
        world = int(os.environ["WORLD_SIZE"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        return rank, world, local
    torch.cuda.set_device(0)
    return 0, 1, 0


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


# ------------------------------------------------------------------------------ reference arm
def cpu_oracle_run(c, A_s: np.ndarray, T_s: np.ndarray, budget_s=20.0):
    """Time the float64 oracle (oracle/) as it stands on the host cores, on a bounded sample of the
    workload: the Gram over the sample matrices (repeated until ~half the budget is spent), one eigh of
    the m x m Gram, and SCW on the sample test matrices; the per-matrix rates are extrapolated to one
    full step (D_train training + D_test test matrices).  Used for the cpu_baseline of our arm's line."""
    import threadpoolctl
    from oracle import scw as oscw
    from oracle import tucker1

    info = threadpoolctl.threadpool_info()
    cores = max([i.get("num_threads", 1) for i in info] + [1])
    G = np.zeros((c.m, c.m))
    nd = 0
    t0 = time.perf_counter()
    while True:
        G += tucker1.mode1_gram(A_s)
        nd += A_s.shape[0]
        if time.perf_counter() - t0 > budget_s * 0.5:
            break
    t_gram = time.perf_counter() - t0
    t0 = time.perf_counter()
    S, lam = tucker1.top_k_eigen(G, c.k)
    t_eig = time.perf_counter() - t0
    t0 = time.perf_counter()
    oscw.scw_errors(T_s, S, c.r)
    t_scw = (time.perf_counter() - t0) / T_s.shape[0]
    t_step = t_gram / nd * c.D_train + t_eig + t_scw * c.D_test
    return {"value": c.D_train / t_step, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"fp64 Gram of {nd} training matrices ({A_s.shape[0]} distinct, {t_gram:.1f}s) + "
                      f"eigh({c.m}) ({t_eig:.2f}s) + SCW of {T_s.shape[0]} test matrices ({t_scw * T_s.shape[0]:.1f}s), "
                      f"rates extrapolated to the full step (D_train={c.D_train}, D_test={c.D_test}); numpy "
                      f"float64 + {info[0].get('internal_api', '?') if info else '?'} BLAS",
            "seconds_per_step": t_step}


def run_reference(args, c):
    """The reference arm = the float64 oracle (the paper has no code to install).  Each timed step is a
    bounded sample of the workload, run for real and reported as timed (no extrapolation): the fp64
    Gram of n_tr training matrices, the top-k eigh of that Gram, and the SCW errors of n_te = n_tr / 4
    test matrices (the 2000 : 500 proportion of C4); value = training matrices per second of that sampled
    pipeline.  n_tr is sized from a probe so that warmup + steps take ~budget seconds in total."""
    import threadpoolctl
    from oracle import scw as oscw
    from oracle import tucker1

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    info = threadpoolctl.threadpool_info()
    cores = max([i.get("num_threads", 1) for i in info] + [1])
    pool_tr = datagen.generate(c, "train", 0, 16).double().numpy()
    pool_te = datagen.generate(c, "test", 0, 4).numpy()
    # probe: seconds per training matrix (Gram), per eigh, per test matrix (SCW)
    t0 = time.perf_counter()
    tucker1.mode1_gram(pool_tr[:2])
    t_mat = (time.perf_counter() - t0) / 2
    t0 = time.perf_counter()
    tucker1.top_k_eigen(np.eye(c.m), c.k)
    t_eig = time.perf_counter() - t0
    t0 = time.perf_counter()
    oscw.scw_errors(pool_te[:1], np.eye(c.m)[: c.k], c.r)
    t_te = time.perf_counter() - t0
    per_step = args.ref_budget / max(1, args.warmup + args.steps)
    n_tr = int(max(4, min(c.D_train, (per_step - t_eig) / (t_mat + t_te / 4))))
    n_te = max(1, n_tr // 4)

    def step():
        idx = np.arange(n_tr) % pool_tr.shape[0]
        G = tucker1.mode1_gram(pool_tr[idx])
        S, lam = tucker1.top_k_eigen(G, c.k)
        oscw.scw_errors(pool_te[np.arange(n_te) % pool_te.shape[0]], S, c.r)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    total = time.perf_counter() - t0
    value = n_tr * args.steps / total
    sample = (f"each step: fp64 Gram of {n_tr} training matrices (cycled from 16 distinct frames) + eigh({c.m}) + "
              f"SCW errors of {n_te} test matrices, timed as run (not extrapolated); numpy float64 + "
              f"{info[0].get('internal_api', '?') if info else '?'} BLAS on {cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (datagen, seed 0)", "config": workload_desc(c, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def run_tsketch(args, c):
    import paper_2209_14637_b200 as tsk
    from paper_2209_14637_b200.dist import init_native_comm, shard_range

    if (args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1) and "NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "INFO"  # init lines on stderr show nranks of the communicators
    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    d0, d1 = shard_range(c.D_train, rank, world)
    t0, t1 = shard_range(c.D_test, rank, world)
    A = datagen.generate(c, "train", d0, d1, device=dev)
    T = datagen.generate(c, "test", t0, t1, device=dev)
    G = torch.empty(c.m, c.m, dtype=torch.float64, device=dev)
    err = torch.empty(t1 - t0, dtype=torch.float64, device=dev)
    ctx = tsk.context(dev)
    if world > 1:
        init_native_comm(ctx)  # the library's own NCCL communicator (tsk_comm_init) for the data path
    stream = torch.cuda.current_stream(dev)
    err_all = torch.empty(c.D_test, dtype=torch.float64, device=dev)
    A_host_sample = A[:8].double().cpu().numpy() if rank == 0 else None
    T_host_sample = T[:2].cpu().numpy() if rank == 0 else None

    ev = {k: [] for k in ("gram", "allreduce", "eig", "scw")}

    def step(record):
        es = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if record else None
        if record:
            es[0].record(stream)
        tsk.sketch_gram(A, G64=G, ctx=ctx)
        if record:
            es[1].record(stream)
        tsk.allreduce_gram(G, ctx=ctx)  # NCCL sum over the ranks (no-op on one GPU)
        if record:
            es[2].record(stream)
        S, lam, info, st = tsk.sketch_topk(G, c.k, ctx=ctx)
        if record:
            es[3].record(stream)
        if t1 > t0:
            tsk.scw_error(T, S, c.r, out=err, ctx=ctx)
        tsk.allgather_errors(err, c.D_test, ctx=ctx)  # every rank's errors -> the whole test set
        if record:
            es[4].record(stream)
        return es, info

    for _ in range(args.warmup):
        step(False)
    barrier(world)
    l0 = ctx.launches
    clocks = clock_sampler(local) if rank == 0 else None
    barrier(world)
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.profiler.start()  # brackets the timed steps for `ncu --profile-from-start off` launch lists
    e_start.record(stream)
    recs = []
    info = None
    for _ in range(args.steps):
        es, info = step(True)
        recs.append(es)
    e_end.record(stream)
    torch.cuda.profiler.stop()
    barrier(world)
    clk = clocks.stop() if clocks else None
    launches = ctx.launches - l0
    total_ms = max_over_ranks(e_start.elapsed_time(e_end), world)
    for es in recs:
        ev["gram"].append(es[0].elapsed_time(es[1]))
        ev["allreduce"].append(es[1].elapsed_time(es[2]))
        ev["eig"].append(es[2].elapsed_time(es[3]))
        ev["scw"].append(es[3].elapsed_time(es[4]))
    phases = {k: max_over_ranks(statistics.mean(v), world) for k, v in ev.items()}
    ms_step = total_ms / args.steps
    value = c.D_train * args.steps / (total_ms / 1e3)

    # ---- end-to-end through the C ABI with HOST buffers (H2D/D2H inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        Ah = torch.empty(tuple(A.shape), dtype=torch.float32, pin_memory=True)
        Ah.copy_(A)
        Th = torch.empty(tuple(T.shape), dtype=torch.float32, pin_memory=True)
        Th.copy_(T)
        Gh = torch.empty(c.m, c.m, dtype=torch.float64).pin_memory()
        errh = torch.empty(t1 - t0, dtype=torch.float64).pin_memory()
        del A
        torch.cuda.empty_cache()

        def e2e_step():
            tsk.sketch_gram(Ah, G64=Gh, ctx=ctx)           # host stack streamed through the library
            if world > 1:
                Gd = Gh.to(dev)
                tsk.allreduce_gram(Gd, ctx=ctx)
                Gh.copy_(Gd)
            S, lam, _, _ = tsk.sketch_topk(Gh, c.k, ctx=ctx)  # host G in, host S out
            if t1 > t0:
                tsk.scw_error(Th, S, c.r, out=errh, ctx=ctx)  # host test stack in, host errors out
            return float(errh.sum()) if t1 > t0 else 0.0

        e2e_step()
        barrier(world)
        tt = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier(world)
        e2e_s = max_over_ranks(time.perf_counter() - tt, world) / args.e2e_steps
        h2d = (d1 - d0) * c.m * c.n * 4 + (t1 - t0) * c.m * c.n * 4 + c.m * c.m * 8 * 2
        d2h = c.m * c.m * 8 * 2 + c.k * c.m * 4 + (t1 - t0) * 8
        e2e = {"value": c.D_train / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "seconds_per_step": e2e_s, "steps": args.e2e_steps,
               "path": "C ABI with pinned host buffers: sketch_gram (H2D streamed, overlapped) -> sketch_topk "
                       "(host G/S) -> scw_error (host tensors)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    mp, peak_kind = measured_peaks()
    derived_tf32 = mp["bf16_tflops_sustained"] * NOMINAL_TF32_OVER_BF16
    # the measured dense TF32 peak of this pool's B200 (scripts/tf32_peak.py: cuBLAS TF32 8192^3, burst and
    # 4 s sustained); the Gram runs ~22 ms per launch at the burst clocks (bench clocks median ~1.9 GHz),
    # so the burst figure is the denominator (the sustained one is taken at power-capped clocks)
    tf32 = None
    try:
        tf32 = json.load(open(os.path.join(ROOT, "profiles", "r02_tf32_peak.json")))
    except Exception:
        tf32 = None
    peak_tf32 = tf32["tf32_tflops_cublas_burst"] if tf32 else derived_tf32
    dloc = d1 - d0
    alg_flops = c.m * (c.m + 1) * c.n * dloc     # lower-triangle Gram, per launch (this rank's shard)
    gram_ms = phases["gram"]
    achieved = alg_flops / (gram_ms / 1e3) / 1e12
    tiles = info.gram_tiles if info and info.gram_tiles else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gram_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == c.name and tj.get("D") == dloc:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # issued tensor-core work of the CTA-pair schedule (gram_pair.cu): 3 products per algorithmic
    # product over the padded 128 x 128 / 128 x 64 pair tiles (a last block with <= 64 valid rows is
    # always the N = 64 B side; an odd tile count adds one dummy half)
    nbk = -(-c.m // 128)
    narrow = (c.m - 128 * (nbk - 1)) <= 64
    t_all = nbk * (nbk + 1) // 2
    t_n64 = nbk if narrow else 0
    t_n128 = t_all - t_n64
    pairs128, pairs64 = -(-t_n128 // 2), -(-t_n64 // 2)
    issued_area = (pairs128 * 2 * 128 * 128 + pairs64 * 2 * 128 * 64) * c.n * dloc * 2 * 3
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf32, "unit": "TFLOP/s",
                "frac": achieved / peak_tf32, "traffic": traffic,
                "kernel": "gram_pair_kernel (tcgen05 cta_group::2, 3xTF32 lower-triangle Gram) + finalize",
                "algorithmic_flops_per_launch": alg_flops,
                "peak_note": (f"TF32 measured on this pool's B200 (profiles/r02_tf32_peak.json, cuBLAS TF32 8192^3): "
                              f"burst {tf32['tf32_tflops_cublas_burst']:.1f}, sustained "
                              f"{tf32['tf32_tflops_cublas_sustained']:.1f} TF/s; burst used (the Gram runs at burst "
                              f"clocks); {peak_kind} bf16 sustained x 1.1/2.25 would give {derived_tf32:.1f}"
                              if tf32 else f"TF32 = {peak_kind} bf16 sustained {mp['bf16_tflops_sustained']} TF/s x "
                              f"nominal 1.1/2.25 (B200_PROFILING.md)"),
                "issued_frac_of_measured_tf32": issued_area / (gram_ms / 1e3) / 1e12 / peak_tf32,
                "issued_tflops": issued_area / (gram_ms / 1e3) / 1e12,
                "issued_frac_of_nominal_tf32": issued_area / (gram_ms / 1e3) / 1.1e15,
                "gram_ms_per_launch": gram_ms}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core products, fp64 partial sums and small solves)",
            "data": f"synthetic (datagen {c.name} recipe, seed 0; paper datasets unavailable)",
            "config": workload_desc(c, world), "phases_ms": phases,
            "sketch_construction_matrices_per_s": c.D_train / ((phases["gram"] + phases["allreduce"] + phases["eig"]) / 1e3),
            "test_matrices_per_s": c.D_test / (phases["scw"] / 1e3) if phases["scw"] > 0 else None,
            "eig_iters": info.iters if info else None, "roofline": roofline, "clocks": clk,
            "gpu_launches": launches, "e2e": e2e}
    if args.cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_oracle_run(c, A_host_sample, T_host_sample, budget_s=args.cpu_budget)
        line["cpu_baseline"].pop("seconds_per_step", None)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tsketch", choices=["tsketch", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=90.0, help="reference arm: seconds for warmup + steps")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    c = datagen.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, c)
    else:
        run_tsketch(args, c)


if __name__ == "__main__":
    main()
