"""Headline benchmark: exact top-K users/sec (f=50, K=10) on the SimDex
index path of BASELINE.json configs[1] (Netflix shape, 480,189 x 17,770,
C=256 k-means with 3 iterations, B=4096 work sharing).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2] [--k K]

One step = exact top-K of every user of the workload through the path the
cost optimizer picks, with the model, clustering and index resident in HBM.
With N ranks (one process per GPU, torchrun) the fixed user set is split
(strong scaling, no data-path collective): the index path routes users by
cluster (sharding.IndexShard), the blocked product cuts contiguous user
blocks (sharding.UserShard), and the catalogue-sharded config (cfg5) splits
the items and exchanges per-user-slice partial lists with an NCCL
all-to-all before the device merge (sharding.CatalogShard).  The time is the
max over ranks.  ``e2e`` is the same metric through the public API from
HOST buffers: upload, cluster, build, estimate, decide, serve, download --
run_pipeline (N = 1) or sharding.run_pipeline_shard (N > 1).

--impl reference times the UNMODIFIED reference package (mipserve, installed
offline into baseline/_ref) on the host cores: P worker processes over
disjoint user samples, one BLAS thread each (the reference protocol,
PAPER.md:1080-1085), each step a bounded sample.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "gemm_topk_traffic.json")
KERNEL_SOURCES = ("paper_1706_01449_b200/csrc/gemm_topk.cu", "paper_1706_01449_b200/csrc/sm100.cuh",
                  "paper_1706_01449_b200/csrc/common.cuh")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--graph", action="store_true", help="(default) replay the serving step as a CUDA graph")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of the graph replay")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def kernel_source_hash():
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        with open(os.path.join(ROOT, rel), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


class Clocks:
    """SM clock and throttle-reason sampling DURING the timed region: an NVML
    thread polling every 2 ms (the timed region of a default run is tens of
    milliseconds, below nvidia-smi's 100 ms loop)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device_index):
        import threading
        self.samples = []
        self.err = None
        self._stop = threading.Event()
        self._on = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device_index]) if vis and vis.split(",")[0].isdigit() else device_index
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = int(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self._reasons = (getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None)
                             or N.nvmlDeviceGetCurrentClocksThrottleReasons)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:  # noqa: BLE001 -- report, do not fail the bench
            self.N, self.err = None, f"nvml unavailable: {e}"

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            if self._on.is_set():
                try:
                    self.samples.append((int(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)),
                                         int(self._reasons(self.h))))
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.002)

    def start_region(self):
        self._on.set()

    def stop(self):
        if self.N is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no sampler"]}
        self._on.clear()
        self._stop.set()
        self.thread.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        reasons = set()
        for _, bits in self.samples:
            for name, attr in self.REASONS:
                if bits & int(getattr(self.N, attr, 0)):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "sampler": "nvml 2 ms"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_path(w):
    return "catalog" if w.name == "cfg5" else w.expected_path


# ---------------------------------------------------------------------------
# the reference package (mipserve, unmodified) on host cores
# ---------------------------------------------------------------------------

_REF = {}


def _import_reference():
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import mipserve
    if not os.path.abspath(mipserve.__file__).startswith(os.path.abspath(REF_PATH)):
        raise ImportError(f"mipserve resolved to {mipserve.__file__}, not baseline/_ref")
    return mipserve


def _import_oracle():
    """The oracle port (oracle/simdex_oracle.py): the stand-in CPU arm when
    baseline/_ref is not installed (bench.py's cpu_baseline / reference arm are
    the only non-test callers of oracle/)."""
    opath = os.path.join(ROOT, "oracle")
    if opath not in sys.path:
        sys.path.insert(0, opath)
    import simdex_oracle
    return simdex_oracle


def _ref_worker(args):
    """One worker's share of a step (reference state inherited through fork)."""
    sample, k = args
    from threadpoolctl import threadpool_limits
    M = _REF["M"]
    with threadpool_limits(1):
        t0 = time.perf_counter()
        if _REF.get("port"):
            users, items = _REF["model"]
            if _REF["index"] is not None:
                M.query_batch(_REF["index"], items, users, sample.tolist(), k, 4096)
            else:
                M.topk_matmul(users[sample], items, k)
        elif _REF["index"] is not None:
            M.query_batch(_REF["index"], _REF["model"], sample.tolist(), k)
        else:
            sub = M.ModelPair(M.FactorMatrix(_REF["model"].users.values[sample]), _REF["model"].items)
            M.topk_matmul(sub, k)
    return len(sample), time.perf_counter() - t0


def reference_setup(w, clustering=None):
    """mipserve model (+ index for the index path).  ``clustering`` = (centroids,
    assignment) to build the reference index from (its own build_index); None
    runs the reference's own kmeans."""
    try:
        M = _import_reference()
    except Exception:  # noqa: BLE001 -- baseline/_ref absent: the oracle port stands in
        O = _import_oracle()
        users, items = w.users.astype(np.float64), w.items.astype(np.float64)
        idx = None
        if w.expected_path == "index":
            if clustering is None:
                cl = O.kmeans(users, w.clusters, max_iters=w.max_iters, seed=w.seed)
                cen, assign, theta = cl["centroids"], cl["assignment"], cl["max_angle"]
            else:
                cen, assign = clustering
                theta = O.compute_max_angles(users, cen, assign)
            ids, bnd, _ = O.build_index(items, cen, theta)
            idx = (ids, bnd, assign)
        _REF.update(M=O, model=(users, items), index=idx, port=True)
        return (users, items), idx
    model = M.ModelPair(M.FactorMatrix(w.users.astype(np.float64)), M.FactorMatrix(w.items.astype(np.float64)))
    idx = None
    if w.expected_path == "index":
        if clustering is None:
            cl = M.kmeans(model.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
        else:
            cen, assign = clustering
            theta = M.compute_max_angles(model.users, M.FactorMatrix(cen), assign)
            c = cen.shape[0]
            cl = M.Clustering(M.FactorMatrix(cen), assign, theta,
                              tuple(np.flatnonzero(assign == j) for j in range(c)), np.empty(0), w.seed)
        idx = M.build_index(model, cl, 4096)
    _REF.update(M=M, model=model, index=idx, port=False)
    return model, idx


def reference_rates(w, k, steps, warmup, cores, per_worker, seed=12345):
    """Per timed step: (users, wall seconds) over `cores` forked workers, each
    on its own random sample of `per_worker` users."""
    import multiprocessing as mp
    rng = np.random.default_rng(seed)
    out = []
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for s in range(warmup + steps):
            samples = [np.sort(rng.choice(w.users.shape[0], per_worker, replace=False)) for _ in range(cores)]
            t0 = time.perf_counter()
            res = pool.map(_ref_worker, [(smp, k) for smp in samples])
            wall = time.perf_counter() - t0
            if s >= warmup:
                out.append((sum(n for n, _ in res), wall))
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1706_01449_b200 import workloads as W
    w = W.CONFIGS[args.config]()
    k = args.k or w.k
    try:
        M = _import_reference()
        kind = "reference"
    except Exception:  # noqa: BLE001 -- the oracle port always exists
        M = None
        kind = "port"
    cores = len(os.sched_getaffinity(0))
    path = workload_path(w)
    t0 = time.perf_counter()
    reference_setup(w)
    setup_s = time.perf_counter() - t0
    per = {"index": 1500, "matmul": 120, "catalog": 2}[path]
    steps = reference_rates(w, k, args.steps, args.warmup, cores, per)
    users = sum(n for n, _ in steps)
    wall = sum(t for _, t in steps)
    v = users / wall
    nu, ni, f = w.users.shape[0], w.items.shape[0], w.users.shape[1]
    what = "query_batch work_sharing=True (B=4096)" if w.expected_path == "index" else "topk_matmul"
    who = (f"mipserve {getattr(M, '__version__', '?')} (baseline/_ref, unmodified)" if kind == "reference"
           else "oracle port (oracle/simdex_oracle.py; baseline/_ref not installed)")
    sample = (f"{who} {what} on {per} random "
              f"users per process per step, {cores} processes x 1 BLAS thread; setup (kmeans + "
              f"build_index) {setup_s:.1f} s, untimed")
    line = {
        "impl": "reference", "metric": f"exact top-K users/sec (f={f}, K={k})", "value": v, "unit": "users/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall / len(steps), "users_per_step": users / len(steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": f"{w.name}: {nu}x{ni}x{f}, K={k}" + (f", C={w.clusters}, B=4096"
                                                                     if w.expected_path == "index" else ""),
                   "path": path},
        "cpu_baseline": {"value": v, "unit": "users/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "users/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_ours(w, k, cl_host):
    """The reference (1 core) on a bounded sample; for the index path its
    index is built by the reference's build_index from the GPU clustering
    (identical to the reference's own k-means at cfg2:
    tests/test_gpu_kernels.py::test_cfg2_full_size_against_reference)."""
    try:
        _, idx = reference_setup(w, cl_host)
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "users/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    per = min(250_000, w.users.shape[0]) if idx is not None else 300  # ~10 s of one core
    steps = reference_rates(w, k, 1, 0, 1, per, seed=777)
    users = sum(n for n, _ in steps)
    wall = sum(t for _, t in steps)
    what = "query_batch work_sharing=True (B=4096)" if idx is not None else "topk_matmul"
    port = bool(_REF.get("port"))
    return {"value": users / wall, "unit": "users/s", "cores": 1, "kind": "port" if port else "reference",
            "sample": f"{'oracle port' if port else 'mipserve'} {what} on {per} random users, 1 process x 1 BLAS "
                      f"thread, {wall:.1f} s"
                      + ("; index by its build_index from the GPU clustering" if idx is not None else ""),
            "cpu_model": cpu_model()}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def committed_traffic(kernel, workload, k, world):
    """DRAM bytes per launch of ``kernel`` from the committed ncu --set full
    capture (profiles/gemm_topk_traffic.json), only when it was taken on the
    current kernel sources (hash match) and on this workload and depth at one
    GPU; else None."""
    try:
        with open(TRAFFIC_FILE) as fh:
            t = json.load(fh)
    except (OSError, ValueError):
        return None, "no committed capture"
    if t.get("kernel_source_hash") != kernel_source_hash():
        return None, "committed capture is from other kernel sources"
    if (t.get("workload", "cfg2"), int(t.get("k", 10))) != (workload, int(k)) or world != 1:
        return None, f"committed capture is of {t.get('workload', 'cfg2')} K={t.get('k', 10)} on one GPU"
    ent = t.get("launches", {}).get(kernel)
    if not ent:
        return None, f"no capture of {kernel}"
    return ent["dram_bytes"], t.get("capture", "")


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1706_01449_b200 as sx
    from paper_1706_01449_b200 import _lib, optimizer, sharding
    from paper_1706_01449_b200 import index as index_mod
    from paper_1706_01449_b200 import workloads as W

    hbm, bf16, peak_kind = peaks()
    w = W.CONFIGS[args.config]()
    k = args.k or w.k
    nu, ni, f = w.users.shape[0], w.items.shape[0], w.users.shape[1]
    model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    dev = torch.device("cuda", local)
    path = workload_path(w)

    # ---- setup (untimed): run_pipeline's stages up to the decision
    setup, decision, est, plan, cl_host, shard, shard_info = {}, None, None, None, None, None, {}
    if path != "catalog":
        plan = optimizer.plan_pipeline(model, k=k, num_clusters=min(w.clusters or 8, nu), block_size=4096,
                                       max_iters=w.max_iters, seed=w.seed)
        decision, est = plan.decision, plan.walk
        setup = {"cluster": plan.cluster_seconds, "build": plan.build_seconds, "estimate": plan.estimate_seconds}
        cl = plan.index.clustering
        cl_host = (cl.centroids.values, np.asarray(cl.assignment))
    served = "catalog" if path == "catalog" else decision  # follow the optimizer
    if served == "index":
        if world > 1:
            shard = sharding.IndexShard(plan.index, model, rank, world, est)
            shard_info = {"users": int(shard.user_ids.size), "work_share": shard.share}

            def step():
                return shard.topk_tensors(k)
        else:
            def step():
                return index_mod.query_batch_tensors(plan.index, model, None, k, work_sharing=True)
    elif served == "matmul":
        if world > 1:
            shard = sharding.UserShard(model, rank, world)
            shard_info = {"users": int(shard.hi - shard.lo)}

        def step():
            return shard.topk_tensors(k) if shard is not None else sx.brute.topk_matmul_tensors(model, k)[:2]
    else:  # catalogue sharded
        if world > 1:
            shard = sharding.CatalogShard(model, rank, world)
            shard_info = {"items": int(shard.model.num_items if shard.model else 0),
                          "users_merged": int(shard.user_hi - shard.user_lo)}

        def step():
            return shard.topk_tensors(k) if shard is not None else sx.brute.topk_matmul_tensors(model, k)[:2]

    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def kernel_pass(fn, steps):
        """per-kernel times: CUDA events recorded by the library on the
        launching stream around each launch, over `steps` eager steps with the
        L2 flushed before each (as in the timed region)"""
        _lib.profile(True)  # (resets the counters)
        for s in range(steps):
            flush.fill_(s & 0x7F)
            fn()
        torch.cuda.synchronize()
        out = {}
        for name in ("gemm_topk", "gemm_topk_prefix", "gemm_topk_full", "finalize", "finalize_prefix",
                     "finalize_full", "walk", "select_rows", "score_f64"):
            ms, n = _lib.profile_read(name)
            if n:
                out[name] = {"ms_per_step": ms / steps, "launches_per_step": n / steps}
        _lib.profile(False)
        return out

    # The serving step is captured once into a CUDA graph and replayed (one
    # host launch per step; --eager times eager launches).  The per-kernel
    # launch times that feed the roofline come from an eager pass of the same
    # number of steps just before the timed region (events cannot be recorded
    # between the kernels of a graph replay).
    graphed = not args.eager and served != "catalog"
    graph_note = None
    kernels = None
    if graphed:
        from paper_1706_01449_b200 import graphs
        for _ in range(args.warmup):
            step()
        kernels = kernel_pass(step, args.steps)
        try:
            n0 = _lib.launch_count()
            step = graphs.GraphedCall(step)
            graph_kernels = (_lib.launch_count() - n0) // 3  # 2 warm-up calls + the captured one
        except Exception as exc:  # noqa: BLE001 -- capture refused: time eager launches instead
            graphed, graph_note, kernels = False, f"graph capture failed ({type(exc).__name__}): eager", None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    if not graphed:
        _lib.profile(True)
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    clocks.start_region()
    for s in range(args.steps):
        flush.fill_(s & 0x7F)
        ev[s][0].record(stream)
        step()
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    if graphed:  # replays launch the captured kernels without host-side counting
        launches = graph_kernels * args.steps
    step_ms = [a.elapsed_time(b) for a, b in ev]
    srt = sorted(step_ms)
    step_stats = {"median": statistics.median(step_ms), "p90": srt[min(len(srt) - 1, int(0.9 * len(srt)))],
                  "min": srt[0], "max": srt[-1]}
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(total_ms.item()) / args.steps
    value = nu / (ms_per_step / 1000.0)  # the fixed user set, all ranks together

    # ---- per-kernel times (eager: recorded during the timed steps)
    if kernels is None:
        kernels = {}
        for name in ("gemm_topk", "gemm_topk_prefix", "gemm_topk_full", "finalize", "finalize_prefix",
                     "finalize_full", "walk", "select_rows", "score_f64"):
            ms, n = _lib.profile_read(name)
            if n:
                kernels[name] = {"ms_per_step": ms / args.steps, "launches_per_step": n / args.steps}
        _lib.profile(False)
    kern_ms = sum(v["ms_per_step"] for name, v in kernels.items() if name.startswith(("gemm", "finalize")))
    roof = roofline(w, k, served, world, kernels, ms_per_step, bf16, peak_kind, _lib,
                    stats=shard.stats() if hasattr(shard, "stats") else None)

    # ---- e2e: public API from host buffers, per step
    e2e = e2e_serve = None
    if not args.no_e2e and served != "catalog":
        e2e = measure_e2e(sx, sharding, model, w, k, served, rank, world, dev, torch, dist)
        e2e_serve = measure_e2e_serve(sx, plan, model, k, served, world, shard, dev, torch, dist, nu)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and served != "catalog":
        cpu = cpu_baseline_ours(w, k, cl_host)

    if rank == 0:
        line = {
            "metric": f"exact top-K users/sec (f={f}, K={k})", "value": value, "unit": "users/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "step_ms": step_stats,
            "main_kernels_ms_per_step": kern_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (exact) / fp16 tensor-core candidates",
            "data": "synthetic (seeded, BASELINE.json shapes; trained Netflix/R2 models unavailable)",
            "config": {"workload": f"{w.name}: {nu}x{ni}x{f}, K={k}" + (f", C={w.clusters}, B=4096"
                                                                         if served == "index" else ""),
                       "path": served, "decision": decision,
                       "mean_visited_sample": None if est is None else est.mean_visited,
                       "parallelism": (f"{world} ranks: " + {"index": "users routed by cluster",
                                                              "matmul": "contiguous user blocks",
                                                              "catalog": "item shards + NCCL all-to-all + merge"}
                                       [served]) if world > 1 else "1 GPU",
                       "rank0_shard": shard_info or None,
                       "l2": "flushed (256 MB write) before every timed step",
                       "launch": ("CUDA graph replay of the serving call (kernel times: eager pass of the same "
                                  "steps before the timed region)") if graphed else (graph_note or "eager"),
                       "setup_seconds": setup},
            "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "e2e_serve": e2e_serve,
            "clocks": clk, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(w, k, served, world, kernels, ms_per_step, bf16, peak_kind, lib, stats=None):
    """Tensor-bound roofline of the dominant kernel, gemm_topk.  Work = 2 f
    flops per (user, item) pair, f unpadded.  Index path: the
    stage-1 prefix launch is the headline and ``frac`` uses SURVEY 8(d)'s
    algorithmic per-unit figure, 2 f B' per user (work sharing scores every
    user's first B' list items); ``frac_executed`` counts only the pairs the
    launch multiplied (simdex_executed_pairs: the prefix early exit skips
    tiles that cannot change the answer).  Both launches and the whole step
    are reported beside it, on executed pairs (the catalogue pass is credited
    with every continuing user x |I|, far above what any exact pass needs).
    Blocked product: every pair is executed unless the norm exit skips tiles;
    ``frac`` counts executed pairs.  Per rank at N > 1 (rank 0)."""
    nu, ni, f = w.users.shape[0], w.items.shape[0], w.users.shape[1]
    peak_note = f"{peak_kind} dense bf16 = fp16 dense rate, burst"
    p1, p2 = lib.executed_pairs()
    if served == "index":
        nq, n_cont, bp, _, _ = lib.ws_stats()
        if stats is not None:  # a rank serving its share as several concurrent calls: their sums
            nq, n_cont, p1, p2 = stats
        s1 = kernels.get("gemm_topk_prefix")
        s2 = kernels.get("gemm_topk_full")
        if not s1:
            return None
        t1 = s1["ms_per_step"] / 1e3
        t12 = t1 + (s2["ms_per_step"] / 1e3 if s2 else 0.0)
        e1, e2 = 2.0 * f * p1, 2.0 * f * p2
        c1, c2 = 2.0 * f * nq * bp, 2.0 * f * n_cont * ni
        traffic, src = committed_traffic("gemm_topk_prefix", w.name, k, world)
        # the algorithmic work of the prefix launch is 2 f B' per
        # user (work sharing scores every user's first B' list items); the
        # early exit skips tiles that cannot change the answer, so the launch
        # multiplies fewer pairs (frac_executed) than it is credited with
        return {"kernel": "gemm_topk_kernel stage 1 (work-sharing prefix: every cluster's first B' list items x "
                          "its users; tcgen05 fp16 -> fp32 TMEM, fused certified top-K)",
                "bound": "tensor", "achieved": c1 / t1 / 1e12, "peak": bf16, "peak_kind": peak_note,
                "unit": "TFLOP/s", "frac": c1 / t1 / 1e12 / bf16, "traffic": traffic, "traffic_source": src,
                "per_unit": f"SURVEY 8(d): 2*f*B' = {2 * f * bp} flop per user (f unpadded), {nq} users per launch; "
                            f"the launch multiplied {p1} of the {nq * bp} credited (user, item) pairs",
                "algorithmic_flops_per_launch": c1, "executed_flops_per_launch": e1, "launch_ms": s1["ms_per_step"],
                "frac_executed": e1 / t1 / 1e12 / bf16,
                "frac_credited": c1 / t1 / 1e12 / bf16,
                "frac_both_launches": (e1 + e2) / t12 / 1e12 / bf16,
                "frac_both_launches_credited": (c1 + c2) / t12 / 1e12 / bf16,
                "both_launches_note": (f"stage 2: {n_cont}/{nq} users continue past B' over |I|={ni}; "
                                       f"{p2} pairs multiplied of {n_cont * ni} credited"),
                "frac_whole_step": (e1 + e2) / (ms_per_step / 1e3) / 1e12 / bf16,
                "share_of_step": s1["ms_per_step"] / ms_per_step}
    g = kernels.get("gemm_topk")
    if not g:
        return None
    if stats is not None:
        p1 = stats[2]
    n_users = nu / world if served == "matmul" else nu
    n_items = ni if served == "matmul" else ni / world
    credited = 2.0 * f * n_items * n_users
    executed = 2.0 * f * p1
    t = g["ms_per_step"] / 1e3
    traffic, src = committed_traffic("gemm_topk", w.name, k, world)
    return {"kernel": "gemm_topk_kernel (blocked product, tcgen05 fp16 -> fp32 TMEM, fused certified top-K)",
            "bound": "tensor", "achieved": executed / t / 1e12, "peak": bf16, "peak_kind": peak_note,
            "unit": "TFLOP/s", "frac": executed / t / 1e12 / bf16, "traffic": traffic, "traffic_source": src,
            "per_unit": f"2*f = {2 * f} flop per multiplied (user, item) pair; {p1} pairs in the launch "
                        f"(credited: 2*f*|I| = {2 * f * ni} per user)",
            "executed_flops_per_launch": executed, "launch_ms": g["ms_per_step"],
            "frac_credited": credited / t / 1e12 / bf16,
            "frac_whole_step": executed / (ms_per_step / 1e3) / 1e12 / bf16,
            "share_of_step": g["ms_per_step"] / ms_per_step}


def measure_e2e(sx, sharding, model, w, k, served, rank, world, dev, torch, dist):
    """run_pipeline from host float64 matrices (pinned H2D inside the timed
    region), results on the host; N > 1: run_pipeline_shard per rank."""
    nu, ni = w.users.shape[0], w.items.shape[0]
    host_u = torch.from_numpy(model.users.values).pin_memory()
    host_i = torch.from_numpy(model.items.values).pin_memory()
    times, rep, n_mine = [], None, nu
    for s in range(8):
        m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        m2.users.__dict__["_device"] = {dev.index: {"f64": host_u.to(dev, non_blocking=True)}}
        m2.items.__dict__["_device"] = {dev.index: {"f64": host_i.to(dev, non_blocking=True)}}
        kw = dict(k=k, num_clusters=min(w.clusters or 8, nu), block_size=4096, max_iters=w.max_iters, seed=w.seed,
                  force=served)
        if world > 1:
            res, rep = sharding.run_pipeline_shard(m2, rank=rank, world=world, **kw)
        else:
            res, rep = sx.run_pipeline(m2, **kw)
        _ = res.item_ids
        n_mine = len(res)
        torch.cuda.synchronize()
        if s >= 2:  # the first passes pay one-time costs (pinned pools, tensor maps, arena growth)
            times.append(time.perf_counter() - t0)
    # median of 6 host-timed passes (a pass is ~20 ms of mostly host-driven
    # orchestration; single passes vary by tens of percent with host noise)
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    k_eff = min(k, ni)
    return {"value": nu / float(t.item()), "unit": "users/s",
            "h2d_bytes_per_step": int(model.users.values.nbytes + model.items.values.nbytes),
            "d2h_bytes_per_step": int(n_mine * (k_eff * (4 + 8) + 8)),
            "passes": len(times), "pass_ms": [round(x * 1e3, 3) for x in times],
            "what": ("run_pipeline" if world == 1 else "sharding.run_pipeline_shard (max over ranks)") +
                    " from host float64 matrices: H2D, k-means, build, estimate, decide, serve, D2H [U,K]",
            "stage_seconds": {"cluster": rep.cluster_seconds, "build": rep.build_seconds,
                              "estimate": rep.estimate_seconds, "serve": rep.serve_seconds}}


def measure_e2e_serve(sx, plan, model, k, served, world, shard, dev, torch, dist, nu):
    """Serving through the public API with the model and index resident:
    query_batch / topk_matmul for every user (this rank's share at N > 1),
    results materialised on the host (D2H inside)."""
    from paper_1706_01449_b200 import _device
    times = []
    d2h = 0
    for s in range(8):  # (the first serves build the per-range query sets and contexts of the overlapped copies)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            out = shard.topk_tensors(k)
            hs = _device.to_host_pinned_many(*out)
            d2h = sum(h.nbytes for h in hs)
        else:
            res = (sx.query_batch(plan.index, model, None, k, work_sharing=True) if served == "index"
                   else sx.topk_matmul(model, k))
            _ = res.item_ids
            d2h = res.item_ids.nbytes + res.scores.nbytes + np.asarray(res.visited).nbytes
        torch.cuda.synchronize()
        if s >= 3:
            times.append(time.perf_counter() - t0)
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"value": nu / float(t.item()), "unit": "users/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": d2h,
            "what": "query_batch / topk_matmul (public API), model + index resident, results to host"}


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
