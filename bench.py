"""Benchmark: MST edges/s for dendrogram construction on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config4]
    python bench.py --impl reference ...        # the reference CPU path (oracle port)

A step = one full `rank_edges + pandora` (the timed scope of `dendromst
build`, cli.py:82-85) over one synthetic MST of BASELINE.json's shape,
inputs resident in HBM: sort of the weights, maxIncident, all contraction
levels, chain walk, chain sort and link.  Default workload = config 4
(random spanning tree n = 128M, tied weights), the configuration the
headline metric is quoted on.  N > 1 runs N independent replicas (one tree
per GPU, no collective on the data path: "replicas only").

`e2e` is the same metric through the public API with HOST buffers: pinned
int32 u, v + float64 w copied in, orig_of / heights / edge_parent /
vertex_parent copied out, every step.
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

METRIC = "MST edges/sec for dendrogram build on 1 B200 (n=128M); % of HBM roofline"
UNIT = "edges/s"

WORKLOADS = {
    # name: (generator, n, description)
    "config4": ("tied", 128_000_000,
                "config4: random spanning tree n=128M, tied weights w in {0..4095} (float64), seed 0"),
    "config4u": ("random", 128_000_000,
                 "config4 companion: random spanning tree n=128M, uniform weights, seed 0"),
    "config3-path": ("path", 16_000_000, "config3: path n=16M, monotone weights (single chain)"),
    "config3-caterpillar": ("caterpillar", 16_000_000,
                            "config3: caterpillar n=16M, monotone weights (single chain)"),
    "random16M": ("random", 16_000_000, "random spanning tree n=16M, uniform weights (config3 reference point)"),
    "config5": ("random", 8_000_000,
                "config5: batch of 64 independent random spanning trees n=8M (uniform weights, seeds 0..63), "
                "tree i on GPU i mod N"),
    "config1": ("random", 100_000, "config1: random spanning tree n=100k, uniform weights, seed 0"),
    "config2": ("blobs1m", 999_999, "config2: EMST of 1M 3-D Gaussian-blob points (mutual reachability, "
                "min_samples=2) computed by the reference, tests/golden/config2_blobs1m.npz"),
}

# Algorithmic HBM bytes of each kernel kind per build: what the
# kernel must read and write given its design, counting a random 4-B access
# as 4 B (the 64-B DRAM sector it really costs is NOT credited; `traffic`
# shows it).  ids / ranks 4 B, weights and keys 8 B (4 B for narrow edge-sort
# keys), records 12 B (maxIncident) or 8 B (chain links).  Which views were
# bucketed and the key width come from the library (dmst_stats path fields),
# not from constants restated here.


def kernel_bytes(stats, n: int, nv: int) -> dict[str, float]:
    counts = stats.view_kind_counts()            # (n_alpha, n_leaf, n_chain, n_k) per view
    info = stats.path_info()
    L = stats.num_levels
    views_n = [c[3] for c in counts]
    views_v = [int(stats.view_vertices[k]) for k in range(L + 1)]
    buck = info["mi_bucketed_views"]             # maxIncident by multisplit + shared-memory apply
    direct = info["mi_direct_views"]             # direct atomics in select_edges, then k_v1
    mb = sum(2 * views_n[k] for k in buck)        # records (2 per edge) of bucketed views
    vb = sum(views_v[k] for k in buck)
    p1, p2 = stats.sort1_passes, stats.sort2_passes
    kb = 4 if info["sort1_narrow"] else 8         # key bytes per item in the edge sort's passes
    item = kb + 12                                # key + (id, u, v) payload
    alpha = sum(c[0] for c in counts[:L])         # edges copied into the next view
    local = info.get("sort1_local") == "smem"     # wide keys: 3 global passes + shared-memory finish
    mids = 2 if local else max(p1 - 2, 0)
    return {
        "sort1_hist": 8.0 * n,                                  # read w
        "sort1_pass_first": (16.0 + item) * n,                  # read w, u, v 16; write key + payload
        "sort1_pass_mid": 2.0 * item * n * mids,                # read + write key + payload per pass
        "sort1_pass_final": 0.0 if local else (item + 20.0) * n,  # read; write orig_of 4, heights 8, euv 8
        "sort1_local": (item + 20.0) * n if local else 0.0,     # read; write orig_of 4, heights 8, euv 8
        "upsweep_scan": float(kb) * n * max(p1 - 1, 0) + 8.0 * n * max(p2 - 1, 0) + 4.0 * n * min(p2, 1),
        "mi_hist": 4.0 * mb,                                    # read endpoints
        "mi_split_a": 16.0 * mb,                                # read 4 + write 12 per record
        "mi_split_b": 24.0 * mb,                                # read 12 + write 12 per record
        "mi_apply": 12.0 * mb + 12.0 * vb,                      # read records; write mi64 8 + parent 4
        "v1": 12.0 * sum(views_v[k] for k in direct),
        "leafscan": 1.0 * sum(views_n),                         # 2-bit counts in, prefixes out (per 16 edges)
        "v2": 12.0 * sum(views_v[1 if info.get("v0_chase") else 0:L]),  # mi64 8 + vertex map 4 (chase hops
                                                                # not credited); view 0 chased in the select: no V2
        "jump": 0.0,
        "select_edges": 9.0 * sum(views_n[:L]) + 4.0 * n + 20.0 * alpha
        + 4.0 * counts[0][2]                                    # view 0's chain edges: x1 gather
        + (4.0 * (counts[0][2] + 2 * counts[0][0]) if info.get("v0_chase") else 0.0)
        + 16.0 * sum(views_n[k] for k in direct),               # euv + ret; x1; alpha: 2 gathers + next view;
                                                                # chased view 0: 8-B maxIncident reads instead
                                                                # of 4-B vertex-map reads (V2's pass dropped);
                                                                # direct views: 2 atomics per next-view edge
        "walk": 17.0 * n,                                       # ret 1 + x1 4 + smi 4 + map 4 + key 4
        "sort2_pass": 16.0 * n * p2,                            # read 8, write 8 per pass
        "link_split": 32.0 * n if p2 else 0.0,                  # two 8-B record passes (read + write)
        "link_apply": 12.0 * n,                                 # read records 8, write edge_parent 4
        "tail": 0.0,                                            # small views (<= 4M edges), L2-resident
        "other": 0.0,
    }


def pipeline_bytes(n: int, S: int) -> int:
    """SURVEY.md §8d byte model: B_alg = 403 n + 98 S, S = sum_{k>=1} n_k."""
    return 403 * n + 98 * S


def load_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    The sampler process is started (and its first line awaited) before the
    region opens; only samples that arrive while the region is open are kept
    (plus the first one after it, so a short region still gets a reading)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.t0 = self.t1 = None

    def start(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.monotonic(), line))
                first.set()
        threading.Thread(target=reader, daemon=True).start()
        first.wait(timeout=10)
        return self

    def __enter__(self):
        if self.proc is None:
            self.start()
        self.t0 = time.monotonic()
        return self

    def __exit__(self, *exc):
        self.t1 = time.monotonic()
        deadline = self.t1 + 0.5
        while time.monotonic() < deadline and not any(t > self.t1 for t, _ in self.lines):
            time.sleep(0.01)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        keep = [ln for t, ln in self.lines if self.t0 is not None and self.t0 <= t <= self.t1]
        after = [ln for t, ln in self.lines if self.t1 is not None and t > self.t1][:1]
        rows = [[p.strip() for p in ln.split(",")] for ln in keep + after]
        rows = [r for r in rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_in_region": len(keep)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


CONFIG5_TREES = 64


def replica_plan(workload: str, world_size: int, rank: int) -> list[int]:
    """Seeds of the trees this rank builds per step.  One tree per GPU
    (seed = rank) for the single-tree workloads ("replicas only": a tree does
    not shard); config 5 deals its 64 trees round-robin,
    tree i -> GPU i mod N."""
    if workload == "config5":
        return [i for i in range(CONFIG5_TREES) if i % world_size == rank]
    return [rank]


def reduce_max(values: list[float], device=None) -> list[float]:
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def reduce_sum(values: list[float], device=None) -> list[float]:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def make_inputs(workload: str, n_override: int | None, seeds: list[int]):
    from paper_2401_06089_b200 import synth
    gen, n, desc = WORKLOADS[workload]
    if n_override:
        n = n_override
    return [synth.GENERATORS[gen](n, seed=sd) for sd in seeds], desc


REF_SITE = os.path.join(ROOT, "baseline", "_ref")   # the unmodified reference, pip-installed


def _import_reference():
    """The unmodified reference package (dendromst) from baseline/_ref, or None."""
    if os.path.isdir(os.path.join(REF_SITE, "dendromst")) and REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "dmst_numba_cache"))
    try:
        import dendromst  # type: ignore
        from dendromst import tree_core  # noqa: F401  (numba import check)
        return dendromst
    except Exception:
        return None


def cpu_worker(args) -> None:
    """Subprocess body: time the reference CPU path exactly as `dendromst
    build` scopes it (cli.py:82-85: perf_counter around rank_edges + pandora)
    on `--n` edges of the workload's shape, `--repeats` times, 1 core.  The
    WeightedTree is built untimed (the inputs are trees by construction; the
    reference's own weighted_tree validation is outside its timed scope too),
    and numba's JIT is warmed on a tiny tree first.  Uses the unmodified
    reference from baseline/_ref when it is installed ("reference"), else the
    oracle port (numpy + C union-find, "port")."""
    from paper_2401_06089_b200 import synth
    gen, _, _ = WORKLOADS[args.workload]
    nv, u, v, w = synth.GENERATORS[gen](args.n, seed=0)
    n = int(u.shape[0])
    R = _import_reference()
    times = []
    if R is not None:
        def mk(nv_, u_, v_, w_):
            k = int(u_.shape[0])
            return R.WeightedTree(int(nv_), np.asarray(u_, np.int64), np.asarray(v_, np.int64),
                                  np.asarray(w_, np.float64), np.arange(k, dtype=np.int64))
        small = synth.random_attach(2000, seed=1)
        R.pandora(R.rank_edges(mk(*small)))
        tree = mk(nv, u, v, w)
        del u, v, w
        for _ in range(args.repeats):
            t0 = time.perf_counter()
            ranked = R.rank_edges(tree)
            R.pandora(ranked)
            times.append(time.perf_counter() - t0)
            del ranked
        try:
            from importlib.metadata import version
            ver = version("dendromst")
        except Exception:
            ver = "?"
        kind, what = "reference", f"unmodified reference dendromst {ver} (baseline/_ref)"
    else:
        from oracle import dendro_oracle as O
        for _ in range(args.repeats):
            t0 = time.perf_counter()
            O.build(nv, u, v, w)
            times.append(time.perf_counter() - t0)
        kind, what = "port", "oracle port of the reference (numpy + C union-find; reference not installed)"
    print(json.dumps({"kind": kind, "what": what, "n": n, "times": times}), flush=True)


def cpu_reference(workload: str, n: int, repeats: int) -> dict:
    """Run cpu_worker in a fresh process (the 128M reference needs ~26 GB of
    host memory, released when it exits)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-worker", "--workload", workload, "--n", str(n),
           "--repeats", str(repeats)]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def reference_sample(n_full: int, steps: int, budget_s: float) -> int:
    """Edges per step for the reference arm: the whole K-step run ~ budget_s
    at the reference's ~0.7e6 edges/s (1 core), between 1M and the full n."""
    per = int(budget_s * 0.7e6 / max(steps, 1))
    return int(min(n_full, max(1_000_000, per // 1_000_000 * 1_000_000)))


def run_reference(args) -> None:
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    _, n_full, desc = WORKLOADS[args.workload]
    n_full = args.n or n_full
    n_sample = args.ref_sample or reference_sample(n_full, args.steps, args.ref_budget)
    r = cpu_reference(args.workload, n_sample, args.steps)
    times = r["times"]
    mean = sum(times) / len(times)
    value = r["n"] / mean
    sample = (f"{r['n']} edges of the {args.workload} shape per step (a bounded sample of the n={n_full} "
              f"workload, sized so K={args.steps} steps take ~{args.ref_budget:.0f} s); {r['what']}; "
              f"rank_edges + pandora timed as cli.py:82-85 scopes it; numba JIT warmed on a 2k-edge tree")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * mean,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int64",
        "data": "synthetic",
        "config": {"workload": desc, "n_edges": n_full, "n_edges_sample_per_step": r["n"],
                   "parallelism": "single core (the reference is single-threaded: numpy + numba without prange)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": r["kind"], "sample": sample,
                         "host_cpus": os.cpu_count(), "times_s": times},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


DIGEST_CASE = {"config4": "config4_tied", "config4u": "config4_uniform", "random16M": "random16M",
               "config3-path": "path16M", "config3-caterpillar": "caterpillar16M", "config2": "config2"}


def reference_parity(workload: str, seeds: list[int], outs) -> dict | None:
    """Compare this run's outputs with the digests of the UNMODIFIED
    reference's outputs on the same inputs (tests/golden/ref_digests/, made by
    tests/golden/make_digests.py): sha256 of int32 orig_of / edge_parent /
    vertex_parent and float64 heights.  Outside the timed region."""
    import hashlib
    ddir = os.path.join(ROOT, "tests", "golden", "ref_digests")
    checked = exact = 0
    for sd, o in zip(seeds, outs):
        case = f"config5_{sd}" if workload == "config5" else (DIGEST_CASE.get(workload) if sd == 0 else None)
        path = os.path.join(ddir, f"{case}.json") if case else None
        if not path or not os.path.exists(path):
            continue
        d = json.load(open(path))
        ok = True
        for key, t, dt in (("orig_of", o.orig_of, np.int32), ("heights", o.heights, np.float64),
                           ("edge_parent", o.edge_parent, np.int32), ("vertex_parent", o.vertex_parent, np.int32)):
            a = np.ascontiguousarray(t.cpu().numpy().astype(dt, copy=False))
            ok &= hashlib.sha256(a.tobytes()).hexdigest() == d[key]
        checked += 1
        exact += int(ok)
    if not checked:
        return None
    return {"trees_checked": checked, "bit_exact": exact,
            "against": "sha256 of the unmodified reference's rank_edges + pandora outputs on the same inputs "
                       "(tests/golden/ref_digests)"}


def run_b200(args) -> None:
    import torch
    ws, rank, local = dist_setup()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from paper_2401_06089_b200 import BuildResult, DendrogramBuilder
    from paper_2401_06089_b200.build import build as build_lib
    if rank == 0:
        build_lib()
    if ws > 1:
        torch.distributed.barrier()

    paths = json.loads(args.paths) if args.paths else None  # code-path overrides (experiments; same results)
    seeds = replica_plan(args.workload, ws, rank)
    trees, desc = make_inputs(args.workload, args.n, seeds)
    n_max = max(int(t[1].shape[0]) for t in trees)
    # several independent trees per GPU run concurrently on S streams (one host
    # thread + builder + workspace each) so one tree's level-loop syncs overlap
    # another tree's kernels
    n_streams = max(1, min(args.streams, len(trees)))
    builders = [DendrogramBuilder(dev) for _ in range(n_streams)]
    for b in builders:
        b.workspace(n_max, n_max + 1)
    streams = [torch.cuda.current_stream(dev)] if n_streams == 1 else \
        [torch.cuda.Stream(device=dev) for _ in range(n_streams)]
    builder = builders[0]
    dev_trees, outs = [], []
    for nv, u, v, w in trees:
        n = int(u.shape[0])
        dev_trees.append((nv, torch.from_numpy(u).to(dev), torch.from_numpy(v).to(dev), torch.from_numpy(w).to(dev)))
        outs.append(BuildResult(orig_of=torch.empty(n, dtype=torch.int32, device=dev),
                                heights=torch.empty(n, dtype=torch.float64, device=dev),
                                edge_parent=torch.empty(n, dtype=torch.int32, device=dev),
                                vertex_parent=torch.empty(nv, dtype=torch.int32, device=dev)))
    edges_rank = sum(int(t[1].shape[0]) for t in trees)
    stream = torch.cuda.current_stream(dev)

    import threading
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=n_streams) if n_streams > 1 else None
    lock = threading.Lock()
    prof: dict[str, list] = {}
    counters = {"launches": 0}
    last_res = [None]

    def run_share(i, profile, start_evt, inputs):
        b, s_ = builders[i], streams[i]
        with torch.cuda.stream(s_):
            if start_evt is not None:
                s_.wait_event(start_evt)
            for t in range(i, len(trees), n_streams):
                nv, du, dv, dw = inputs[t]
                res = b.build(nv, du, dv, dw, out=outs[t], profile=profile, paths=paths)
                last_res[0] = res
                with lock:
                    counters["launches"] += int(res.stats.kernel_launches)
                if profile:
                    with lock:
                        for k, (ms, calls) in res.stats.kernel_profile().items():
                            p = prof.setdefault(k, [0.0, 0])
                            p[0] += ms
                            p[1] += calls
            done = torch.cuda.Event()
            done.record(s_)
        return done

    def step(profile=False, inputs=None):
        inputs = inputs or dev_trees
        cur = torch.cuda.current_stream(dev)
        start = torch.cuda.Event()
        start.record(cur)
        if pool is None:
            done = [run_share(0, profile, start, inputs)]
        else:
            done = list(pool.map(lambda i: run_share(i, profile, start, inputs), range(n_streams)))
        for d in done:
            cur.wait_event(d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    counters["launches"] = 0

    # ---------------- device-resident timed region ----------------
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev.index).start()
    with clk:
        e0.record(stream)
        # per-kernel CUDA events bracket every launch of the LAST timed step
        # only (event records cost ~0.6 ms of host time per build, which
        # would otherwise be charged to every step)
        for i in range(args.steps):
            step(profile=i == args.steps - 1)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    launches = counters["launches"]
    res = last_res[0]
    ms_step = e0.elapsed_time(e1) / args.steps
    stats = res.stats
    counts = stats.view_kind_counts()
    n_last = int(dev_trees[-1][1].shape[0])
    S = sum(c[3] for c in counts[1:])

    parity = reference_parity(args.workload, seeds, outs) if not args.n else None
    chk = reduce_sum([float(parity["trees_checked"]) if parity else 0.0,
                      float(parity["bit_exact"]) if parity else 0.0], device=dev)  # every rank joins
    parity = {"trees_checked": int(chk[0]), "bit_exact": int(chk[1]),
              "against": "sha256 of the unmodified reference's rank_edges + pandora outputs on the same inputs "
                         "(tests/golden/ref_digests)"} if chk[0] else None

    # ---------------- end-to-end through the public API (host buffers) ----------------
    # DendrogramBuilder.build_host (C ABI dmst_build_host): pinned host
    # inputs copied in, every output copied back to pinned host buffers as
    # soon as its stage is done, all inside the timed region.  `depth` builds
    # are in flight at once (one host thread + stream + workspace each), so
    # one build's copies overlap another's kernels (PCIe is full duplex);
    # depth 1 is reported too ("serial").
    from paper_2401_06089_b200 import HostBuildResult
    host_in = [(nv, torch.from_numpy(u).pin_memory(), torch.from_numpy(v).pin_memory(),
                torch.from_numpy(w).pin_memory()) for nv, u, v, w in trees]
    del builders, pool, builder
    torch.cuda.empty_cache()
    depth = max(1, args.e2e_depth)
    e2e_workers = max(depth, n_streams)
    e2e_builders = [DendrogramBuilder(dev) for _ in range(e2e_workers)]
    for b in e2e_builders:
        b.host_workspace(n_max, n_max + 1)
    e2e_streams = [torch.cuda.Stream(device=dev) for _ in range(e2e_workers)]
    e2e_outs = [HostBuildResult.empty(n_max, n_max + 1) for _ in range(e2e_workers)]
    e2e_pool = ThreadPoolExecutor(max_workers=e2e_workers)

    def e2e_run(n_steps: int, workers: int) -> float:
        """n_steps steps (each: every tree of this rank once) on `workers`
        concurrent builders; returns device ms per step (CUDA events)."""
        jobs = [(s_i, t) for s_i in range(n_steps) for t in range(len(trees))]

        def work(i, start_evt):
            b, s_ = e2e_builders[i], e2e_streams[i]
            with torch.cuda.stream(s_):
                s_.wait_event(start_evt)
                for _, t in jobs[i::workers]:
                    nv, hu, hv, hw = host_in[t]
                    n_t = int(hu.shape[0])
                    o = e2e_outs[i]
                    b.build_host(nv, hu, hv, hw, paths=paths, out=HostBuildResult(
                        o.orig_of[:n_t], o.heights[:n_t], o.edge_parent[:n_t], o.vertex_parent[:nv]))
                done = torch.cuda.Event()
                done.record(s_)
            return done

        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        done = list(e2e_pool.map(lambda i: work(i, f0), range(workers)))
        for d in done:
            stream.wait_event(d)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        return f0.elapsed_time(f1) / n_steps

    e2e_steps = max(2, args.e2e_steps)
    e2e_run(depth, depth)  # warm-up
    e2e_ms = e2e_run(e2e_steps, depth)
    e2e_serial_ms = e2e_run(max(1, e2e_steps // 2), 1) if depth > 1 else e2e_ms
    he0 = e2e_outs[0].edge_parent
    n0 = int(dev_trees[0][1].shape[0])
    if len(trees) == 1 and not np.array_equal(he0[:n0].numpy(), outs[0].edge_parent.cpu().numpy()):
        raise RuntimeError("e2e output mismatch")

    # ---------------- input validation (not in the timed scope) ----------------
    from paper_2401_06089_b200.api import _validate
    nv0, du0, dv0, dw0 = dev_trees[0]
    vb = e2e_builders[0]
    _validate(vb, nv0, du0, dv0, dw0)
    vtimes = []
    for _ in range(3):
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(torch.cuda.current_stream(dev))
        _validate(vb, nv0, du0, dv0, dw0)
        g1.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        vtimes.append(g0.elapsed_time(g1))
    validate_ms = statistics.median(vtimes)

    # ---------------- max over ranks (time), sum over ranks (work) ----------------
    ms_step, e2e_ms, e2e_serial_ms = reduce_max([ms_step, e2e_ms, e2e_serial_ms], device=dev)
    (edges_total,) = reduce_sum([float(edges_rank)], device=dev)
    h2d = sum(int(t[1].shape[0]) * 16 for t in trees)
    d2h = sum(int(t[1].shape[0]) * 16 + int(t[0]) * 4 for t in trees)
    h2d, d2h = reduce_sum([float(h2d), float(d2h)], device=dev)

    if rank == 0:
        peak, peak_src = load_peaks()
        # every kernel kind: algorithmic bytes / device time over the timed
        # region (CUDA events on the launching stream); the dominant kind
        # (largest device time) is the headline `roofline`
        per_build = kernel_bytes(stats, n_last, n_last + 1)
        builds = len(trees)  # profiled: the last timed step
        traffic_tab = {}
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic_tab = json.load(open(tpath)).get(args.workload, {})
            except Exception:
                traffic_tab = {}
        kroof = {}
        for k, (kms, kcalls) in prof.items():
            bts = per_build.get(k, 0.0) * builds
            kroof[k] = {"ms_per_build": kms / builds, "launches_per_build": kcalls / builds,
                        "algorithmic_bytes_per_build": bts / builds,
                        "achieved_GBs": bts / (kms * 1e-3) / 1e9 if kms > 0 else 0.0}
        kname, (kms, kcalls) = max(prof.items(), key=lambda kv: kv[1][0])
        kr = kroof[kname]
        roof = {"bound": "hbm", "kernel": kname, "achieved": kr["achieved_GBs"], "peak": peak, "unit": "GB/s",
                "frac": kr["achieved_GBs"] / peak, "traffic": traffic_tab.get(kname),
                "algorithmic_bytes_per_launch": kr["algorithmic_bytes_per_build"] / max(kr["launches_per_build"], 1e-9),
                "avg_launch_ms": kms / kcalls, "launches_per_build": kr["launches_per_build"],
                "peak_source": peak_src,
                "note": "traffic = ncu dram__bytes_read+write per launch (profiles/ncu_traffic.json)"}
        if roof["traffic"]:
            # what the DRAM actually moved for this kind (random 4-8 B accesses cost 64-B
            # sectors), per launch over the live launch time: how close it runs to the wall
            roof["dram_frac"] = roof["traffic"] / (roof["avg_launch_ms"] * 1e-3) / 1e9 / peak
        B = sum(pipeline_bytes(int(t[1].shape[0]), S) for t in trees) * ws
        pipe_ach = B / (ms_step * 1e-3) / 1e9
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            n_s = min(args.cpu_sample or n_last, n_last)
            r = cpu_reference(args.workload, n_s, args.cpu_repeats)
            cpu = {"value": r["n"] / statistics.median(r["times"]), "unit": UNIT, "cores": 1, "kind": r["kind"],
                   "sample": (f"{'the full workload' if r['n'] == n_last else 'a bounded sample'}: {r['n']} edges "
                              f"of the {args.workload} shape, median of {len(r['times'])} run(s) "
                              f"({', '.join(f'{t:.1f}' for t in r['times'])} s); {r['what']}; rank_edges + pandora "
                              f"timed as cli.py:82-85 scopes it, 1 core"),
                   "host_cpus": os.cpu_count(), "host_affinity": len(os.sched_getaffinity(0))}
        n_tree = n_last
        line = {
            "metric": METRIC, "value": edges_total / (ms_step * 1e-3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.workload != "config5" else "strong",
            "vs_baseline": None, "dtype": "u64-key+int32", "data": "synthetic",
            "config": {"workload": desc, "n_edges": n_tree, "n_vertices": n_tree + 1,
                       "streams_per_gpu": n_streams,
                       "trees_per_step": len(seeds) * ws if args.workload != "config5" else CONFIG5_TREES,
                       "per_gpu": (f"{len(seeds)} tree(s) on rank 0; independent trees per GPU, no collective"),
                       "l2": "inputs (16 B/edge = %.1f GB) and working set larger than the 126 MB L2"
                             % (16 * n_tree / 1e9) if n_tree > 10_000_000 else "working set per tree vs 126 MB L2",
                       "parallelism": f"replicas x{ws}", "levels": stats.num_levels,
                       "paths": stats.path_info(), "S_over_n": S / n_tree},
            "e2e": {"value": edges_total / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
                    "api": "DendrogramBuilder.build_host -> dmst_build_host (pinned host buffers)",
                    "builds_in_flight": depth, "builds_timed": e2e_steps,
                    "serial": {"value": edges_total / (e2e_serial_ms * 1e-3), "ms_per_step": e2e_serial_ms,
                               "builds_in_flight": 1}},
            "roofline": roof,
            "validation": {"ms": validate_ms, "edges_per_s": int(dev_trees[0][1].shape[0]) / (validate_ms * 1e-3),
                           "what": "weighted_tree checks (tree_core.py:110-139) on the device, valid input: "
                                   "one scan + lock-free union-find; outside the timed build scope like the reference"},
            "pipeline_roofline": {"bound": "hbm", "achieved": pipe_ach, "peak": peak, "unit": "GB/s",
                                  "frac": pipe_ach / peak, "algorithmic_bytes_per_step": B,
                                  "model": "403 n + 98 S (SURVEY.md 8d)", "peak_source": peak_src,
                                  "frac_vs_nominal_8TBs": pipe_ach / 8000.0},
            "kernel_ms_per_step": {k: v[0] for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
            "kernel_profile": "CUDA events around every launch of the last of the K timed steps",
            "kernel_roofline": {k: {"ms": round(v["ms_per_build"], 4), "GBs": round(v["achieved_GBs"], 1),
                                    "frac": round(v["achieved_GBs"] / peak, 4)}
                                for k, v in sorted(kroof.items(), key=lambda kv: -kv[1]["ms_per_build"])},
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="config4")
    ap.add_argument("--n", type=int, default=None, help="override the workload's edge count")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="edges for cpu_baseline (0 = the full workload tree; 128M takes ~4 min)")
    ap.add_argument("--cpu-repeats", type=int, default=1)
    ap.add_argument("--streams", type=int, default=8, help="concurrent trees per GPU (multi-tree workloads)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="reference arm: edges per step (0 = sized by --ref-budget)")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="reference arm: seconds for all K steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--paths", default="", help="JSON dmst_stats path overrides, e.g. '{\"sort2_geometry\": 4}'")
    ap.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--repeats", type=int, default=1, help=argparse.SUPPRESS)
    ap.add_argument("--e2e-depth", type=int, default=2, help="builds in flight in the e2e leg")
    ap.add_argument("--e2e-steps", type=int, default=12,
                    help="builds timed in the e2e leg (a stream of builds: pipeline fill and drain included)")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("bad steps/warmup")
    if args.cpu_worker:
        cpu_worker(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
