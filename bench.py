"""Headline benchmark: exact top-K users/sec (f=50, K=10) on the SimDex
index path of BASELINE.json configs[1] (Netflix shape, 480,189 x 17,770,
C=256 k-means with 3 iterations, B=4096 work sharing).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One step = serve every user of the workload (exact top-K, the path the
cost optimizer picks) with the model, clustering and index already resident
in HBM.  Each rank of an N-GPU run serves its own full copy of the workload
(weak scaling, no data-path collective).  ``e2e`` is the same metric through
the public API from HOST buffers: upload (pinned), cluster, build, estimate,
decide, serve, download the [U, K] results -- i.e. run_pipeline.

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, the reference being pure Python) on the host cores,
P worker processes over disjoint user slices, each step a bounded sample.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.path = f"/tmp/simdex_clocks_{os.getpid()}.csv"
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.skip = 0

    def _rows(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7 and parts[0].isdigit():
                    rows.append(parts)
        except OSError:
            pass
        return rows

    def start_region(self):
        """Wait (<= 5 s) until the sampler is producing, then mark the start of
        the timed region: only samples taken after this point are reported."""
        if self.proc is None:
            return
        t0 = time.time()
        while not self._rows() and time.time() - t0 < 5.0:
            time.sleep(0.02)
        self.skip = len(self._rows())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = self._rows()[self.skip:]
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[0]) for r in rows]
        reasons = set()
        for r in rows:
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]), "reasons": sorted(reasons),
                "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: the oracle port on host cores
# ---------------------------------------------------------------------------

_CPU_STATE = {}


def _cpu_worker(args):
    """One worker's share of a step (state inherited through fork)."""
    sample, k, block = args
    import simdex_oracle as O
    st = _CPU_STATE
    t0 = time.perf_counter()
    O.query_batch(st["index"], st["items"], st["users"], list(sample), k, block)
    return len(sample), time.perf_counter() - t0


def cpu_reference(workload, k, steps, warmup, cores, per_worker, block=4096, matmul=False):
    """Time the reference algorithm (oracle port) on `cores` processes; returns
    (users/s per step list, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import multiprocessing as mp

    import simdex_oracle as O
    users = workload.users.astype(np.float64)
    items = workload.items.astype(np.float64)
    rng = np.random.default_rng(12345)
    if matmul:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)

        def one(sample):
            t0 = time.perf_counter()
            O.topk_matmul(users[sample], items, k)
            return len(sample), time.perf_counter() - t0
        rates = []
        for s in range(warmup + steps):
            sample = np.sort(rng.choice(users.shape[0], per_worker, replace=False))
            n, dt = one(sample)
            if s >= warmup:
                rates.append(n / dt)
        return rates, f"topk_matmul on {per_worker} random users per step, 1 process"
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)  # the reference protocol: one BLAS thread per process
    cl = O.kmeans(users, workload.clusters, workload.max_iters, workload.seed)
    ids, bounds, _ = O.build_index(items, cl["centroids"], cl["max_angle"])
    _CPU_STATE.update(index=(ids, bounds, cl["assignment"]), items=items, users=users)
    rates = []
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for s in range(warmup + steps):
            samples = [np.sort(rng.choice(users.shape[0], per_worker, replace=False)) for _ in range(cores)]
            t0 = time.perf_counter()
            out = pool.map(_cpu_worker, [(smp, k, block) for smp in samples])
            wall = time.perf_counter() - t0
            if s >= warmup:
                rates.append(sum(n for n, _ in out) / wall)
    return rates, (f"query_batch work-sharing (B={block}) over {per_worker} random users per process per step, "
                   f"{cores} processes, index built by the oracle k-means/build_index")


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1706_01449_b200 import workloads as W
    w = W.CONFIGS[args.config]()
    k = args.k or w.k
    cores = len(os.sched_getaffinity(0))
    matmul = w.expected_path == "matmul"
    per = 400 if matmul else 2000
    rates, sample = cpu_reference(w, k, args.steps, args.warmup, cores, per, matmul=matmul)
    v = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": f"exact top-K users/sec (f={w.users.shape[1]}, K={k})", "value": v,
        "unit": "users/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * w.users.shape[0] / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": f"{w.name}: {w.users.shape[0]}x{w.items.shape[0]}x{w.users.shape[1]} K={k}",
                   "path": "matmul" if matmul else "index+work-sharing"},
        "cpu_baseline": {"value": v, "unit": "users/s", "cores": 1 if matmul else cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "users/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _profiled_traffic(path, k):
    """DRAM bytes per gemm_topk launch (read + write) from the committed ncu
    --set full capture of the same workload (profiles/), or None."""
    f = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01h_gemm_topk_traffic.json")
    if path != "index" or k != 10 or not os.path.exists(f):
        return None
    with open(f) as fh:
        return json.load(fh)["traffic_bytes_per_launch"]


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1706_01449_b200 as sx
    from paper_1706_01449_b200 import _device, _lib, _ops, optimizer
    from paper_1706_01449_b200 import index as index_mod
    from paper_1706_01449_b200 import workloads as W

    hbm, bf16, peak_kind = peaks()
    w = W.CONFIGS[args.config]()
    k = args.k or w.k
    nu, ni, f = w.users.shape[0], w.items.shape[0], w.users.shape[1]
    model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    dev = torch.device("cuda", local)

    # ---- setup (untimed): cluster, build, estimate, decide -- run_pipeline's stages
    t0 = time.perf_counter()
    cl = sx.kmeans(model.users, min(w.clusters or 8, nu), max_iters=w.max_iters, seed=w.seed)
    torch.cuda.synchronize()
    t_cluster = time.perf_counter() - t0
    t0 = time.perf_counter()
    idx = sx.build_index(model, cl, 4096)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    est = sx.estimate_walk_length(idx, model, 0.001, k, seed=w.seed)
    decision = sx.decide(est.mean_visited, ni, 4096, k, optimizer.resolve_h0(None))
    path = w.expected_path if args.config != "cfg2" else decision
    q = torch.arange(nu, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)  # > 126 MB L2

    if path == "index":
        def step():
            return index_mod.query_batch_tensors(idx, model, None, k, work_sharing=True)
    else:
        def step():
            return sx.brute.topk_matmul_tensors(model, k)

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start_region()
    _lib.profile(True)
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for s in range(args.steps):
        flush.fill_(s & 0x7F)
        ev[s][0].record(stream)
        out = step()
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    step_sorted = sorted(step_ms)
    step_stats = {"median": statistics.median(step_ms), "p90": step_sorted[min(len(step_sorted) - 1,
                                                                              int(0.9 * len(step_sorted)))],
                  "min": step_sorted[0], "max": step_sorted[-1]}
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(total_ms.item()) / args.steps
    value = world * nu / (ms_per_step / 1000.0)

    # ---- dominant kernel roofline: per-kernel CUDA events recorded by the
    # library on the launching stream during the timed steps (simdex_profile_*)
    kernels = {}
    for name in ("gemm_topk", "finalize", "walk", "select_rows", "score_f64"):
        ms, n = _lib.profile_read(name)
        if n:
            kernels[name] = {"ms_per_step": ms / args.steps, "launches_per_step": n / args.steps}
    _lib.profile(False)
    gemm_ms = kernels.get("gemm_topk", {}).get("ms_per_step")
    k_eff = min(k, ni)
    if path == "index":
        # two tensor-core passes per step: every user x its cluster's first B'
        # list items, then the users not certified at B' x the whole catalogue
        nq, n_cont, bp, _, _ = _lib.ws_stats()
        flops = 2.0 * f * (nq * bp + n_cont * ni)
        per_unit = (f"2*f*(B' + frac_continuing*|I|) flop per user: B'={bp}, continuing {n_cont}/{nq} users "
                    f"({n_cont / max(nq, 1):.3f}) over |I|={ni}")
    else:
        flops = 2.0 * f * ni * nu
        per_unit = f"2*f*|I| = {2 * f * ni} flop per user"
    roof = None
    if gemm_ms:
        achieved = flops / (gemm_ms / 1000.0) / 1e12
        roof = {"kernel": "gemm_topk_kernel (tcgen05 fp16 x fp16 -> fp32 TMEM, fused certified top-K)",
                "bound": "tensor", "achieved": achieved, "peak": bf16, "peak_kind": f"{peak_kind} dense bf16 (= fp16 dense rate on B200; burst)",
                "unit": "TFLOP/s", "frac": achieved / bf16, "traffic": _profiled_traffic(path, k),
                "algorithmic_flops_per_step": flops, "launch_ms_per_step": gemm_ms,
                "launches_per_step": kernels["gemm_topk"]["launches_per_step"], "per_unit": per_unit,
                "share_of_step": gemm_ms / ms_per_step,
                # BASELINE's north star states its GEMM target against a split-fp32
                # peak (3xTF32 = dense bf16 / 6 with TF32 = bf16 / 2); the certified
                # single-pass fp16 product needs one pass, so it can exceed that
                "split_fp32_peak": bf16 / 6.0, "frac_vs_split_fp32_peak": achieved / (bf16 / 6.0)}

    # ---- e2e: public API from host buffers (run_pipeline), per step
    e2e = None
    if not args.no_e2e:
        host_u = torch.from_numpy(model.users.values).pin_memory()
        host_i = torch.from_numpy(model.items.values).pin_memory()
        e2e_steps = max(1, min(3, args.steps))
        e2e_warm = 2  # first passes pay one-time costs (pinned host pools, tensor maps, allocator growth)
        times = []
        for s in range(e2e_steps + e2e_warm):
            m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m2.users.__dict__["_device"][local] = {"f64": host_u.to(dev, non_blocking=True)}
            m2.items.__dict__["_device"][local] = {"f64": host_i.to(dev, non_blocking=True)}
            res, rep = sx.run_pipeline(m2, k=k, num_clusters=min(w.clusters or 8, nu), block_size=4096,
                                       max_iters=w.max_iters, seed=w.seed, force=path)
            _ = res.item_ids  # results are host arrays [U, K] once run_pipeline returns
            torch.cuda.synchronize()
            if s >= e2e_warm:
                times.append(time.perf_counter() - t0)
        t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        k_eff = min(k, ni)
        e2e = {"value": world * nu / float(t.item()), "unit": "users/s",
               "h2d_bytes_per_step": int(model.users.values.nbytes + model.items.values.nbytes),
               "d2h_bytes_per_step": int(nu * k_eff * (4 + 8) + nu * 8),
               "what": "run_pipeline from host float64 matrices: H2D, k-means, build, estimate, serve, D2H [U,K]",
               "stage_seconds": {"cluster": rep.cluster_seconds, "build": rep.build_seconds,
                                 "estimate": rep.estimate_seconds, "serve": rep.serve_seconds}}

    # ---- serving through the public API with the model and index resident:
    # query_batch for every user, results materialised on the host (D2H inside)
    e2e_serve = None
    if not args.no_e2e:
        times = []
        for s in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if path == "index":
                res = sx.query_batch(idx, model, None, k, work_sharing=True)
            else:
                res = sx.topk_matmul(model, k)
            _ = res.item_ids
            torch.cuda.synchronize()
            if s >= 1:
                times.append(time.perf_counter() - t0)
        t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_serve = {"value": world * nu / float(t.item()), "unit": "users/s", "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": int(nu * min(k, ni) * (4 + 8) + nu * 8),
                     "what": "query_batch (public API) for all users, model + index resident, results to host"}

    # ---- CPU baseline (rank 0, N=1 only): the reference algorithm on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        matmul = path == "matmul"
        rates, sample = cpu_reference(w, k, 2, 0, 1, 300 if matmul else 8000, matmul=matmul)
        cpu = {"value": float(np.mean(rates)), "unit": "users/s", "cores": 1, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": f"exact top-K users/sec (f={f}, K={k})", "value": value, "unit": "users/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (exact) / fp16 tensor-core candidates",
            "data": "synthetic (seeded, BASELINE.json shapes; trained Netflix/R2 models unavailable)",
            "config": {"workload": f"{w.name}: {nu}x{ni}x{f}, K={k}, C={cl.num_clusters}, B=4096",
                       "path": path, "decision": decision, "mean_visited_sample": est.mean_visited,
                       "per_rank_users": nu, "parallelism": f"users-dp{world} (each rank serves the full batch)",
                       "l2": "flushed (256 MB write) before every timed step",
                       "setup_seconds": {"cluster": t_cluster, "build": t_build}},
            "step_ms": step_stats, "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "e2e_serve": e2e_serve, "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
