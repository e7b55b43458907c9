"""Flood-filtration benchmark (BASELINE.json metric: simplices/s).

One step = one GPU pass of the hot path over the workload with the cloud and
the landmark complex resident in HBM: spatial-grid build, the flooding
kernel for every simplex of dim <= max_dim, facet completion.  The default
workload is BASELINE configs[1]: 1M points, noisy sphere+torus mix, 2000
FPS landmarks, simplices of dim <= 2 of their 3-D Delaunay complex, grid
resolution m = 20 (the reference default).  Farthest point sampling and the
host Delaunay are timed as separate stages (fps_ms, delaunay_s); fps_ms has
the CPU oracle's time beside it (fps_cpu_baseline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config sphere_torus_1m|dense30_1m|box_10m|torus_10k|modelnet_batch]

Single-cloud configs at N > 1 (torchrun): every rank builds the grid, values
an interleaved shard of the simplices, and the shards are all-gathered over
NCCL ("scaling": "strong", the complex is fixed).  modelnet_batch (configs[3])
gives every rank its own 64 clouds ("scaling": "weak"; 512 clouds at N = 8):
the step values all of them, no collective.
--impl reference times the CPU oracle (oracle/, a C restatement of the
reference algorithm, all host threads) on a bounded sample of the same
complex; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, n_points, landmarks, m, max_dim)
    "sphere_torus_1m": ("sphere_torus", 1_000_000, 2000, 20, 2),
    "dense30_1m": ("sphere_torus", 1_000_000, 2000, 30, 2),
    "box_10m": ("box", 10_000_000, 5000, 20, 3),
    "torus_10k": ("torus", 10_000, 500, 20, 2),
    "modelnet_batch": ("modelnet", 100_000, 1000, 20, 3),
}
BATCH_PER_RANK = 64  # modelnet_batch: clouds per GPU (512 over 8 GPUs)


def _cloud(kind: str, n: int, seed: int = 0):
    from paper_2509_22432_b200 import datagen

    if kind == "sphere_torus":
        return datagen.gen_sphere_torus_mix(n, seed=seed).points
    if kind == "box":
        return datagen.gen_uniform_box(n, seed=seed).points
    if kind == "modelnet":
        return datagen.gen_modelnet_like(n, seed=seed).points
    return datagen.gen_torus(n, seed=seed).points


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in
    process through NVML (initialised before the region starts): spawning
    nvidia-smi inside the region stalled kernel launches -- an eager box_10m
    step read ~2x slow whenever a spawn landed in it.  Falls back to
    nvidia-smi when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period: float = 0.05):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        self._h = None

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
        r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        flags = [n.nvmlClocksEventReasonHwSlowdown, n.nvmlClocksEventReasonHwThermalSlowdown,
                 n.nvmlClocksEventReasonSwThermalSlowdown, n.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx)] + ["Active" if r & f else "Not Active" for f in flags]

    def _sample_smi(self):
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            return [c.strip() for c in out.stdout.strip().split(",")]
        return None

    def _run(self):
        while not self._stop.is_set():
            try:
                row = self._sample_nvml() if self._nvml is not None else self._sample_smi()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            self._stop.wait(self.period if self._nvml is not None else 0.2)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            try:  # the CUDA device's own GPU (NVML indices ignore CUDA_VISIBLE_DEVICES)
                import torch

                pr = torch.cuda.get_device_properties(self.index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml = pynvml
        except Exception:
            self._nvml = None
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        if self._nvml is not None:
            try:
                self._nvml.nvmlShutdown()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def prepare(cfg_name: str, device: int, rank: int = 0):
    """Untimed setup: clouds, GPU FPS (timed as its own stage), host Delaunay,
    device complexes.  Batch configs hold this rank's BATCH_PER_RANK clouds."""
    import torch

    from paper_2509_22432_b200 import farthest_point_sampling, farthest_point_sampling_batched
    from paper_2509_22432_b200.batch import DeviceComplex
    from paper_2509_22432_b200.delaunay import delaunay

    kind, n, nl, m, max_dim = CONFIGS[cfg_name]
    batch = kind == "modelnet"
    dev = torch.device(f"cuda:{device}")
    if batch:
        seeds = [rank * BATCH_PER_RANK + i for i in range(BATCH_PER_RANK)]
        Xs = [_cloud(kind, n, s) for s in seeds]
        Xd = torch.from_numpy(np.stack(Xs)).to(dev)
        fps = lambda: farthest_point_sampling_batched(Xd, nl, 0)  # noqa: E731
    else:
        Xs = [_cloud(kind, n)]
        Xd = torch.from_numpy(Xs[0]).to(dev)
        fps = lambda: farthest_point_sampling(Xd, nl, 0).reshape(1, -1)  # noqa: E731
    fps()  # warm the FPS kernel
    torch.cuda.synchronize()
    fps_ms = []
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = fps()
        e1.record()
        torch.cuda.synchronize()
        fps_ms.append(e0.elapsed_time(e1))
    idx = idx.cpu().numpy()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        tris = list(pool.map(lambda i: delaunay(Xs[i][idx[i]]), range(len(Xs))))
    delaunay_s = time.perf_counter() - t0
    items = []
    for i, tri in enumerate(tris):
        dc = DeviceComplex(tri, dev, max_dim)
        items.append((Xd[i] if batch else Xd, dc))
    top = min(max_dim, tris[0].dim)
    return dict(X=Xs[0], Xs=Xs, Xd=Xd, idx=idx[0], idxs=idx, tri=tris[0], tris=tris, m=m,
                max_dim=top, n=n, nl=nl, fps_ms=min(fps_ms), delaunay_s=delaunay_s, kind=kind,
                items=items, batch=batch, dev=dev)


def step_single(lib, native, w, stream):
    """One cloud in one fph_flood_filtration call; a batch's clouds one call
    each, on two streams forked from `stream` (two in flight)."""
    from paper_2509_22432_b200.batch import flood_sq_device, flood_sq_device_many

    if len(w["items"]) == 1:
        Xd, dc = w["items"][0]
        flood_sq_device(Xd, dc, w["m"], True, stream)
    else:
        flood_sq_device_many(w["items"], w["m"], True, stream,
                             lanes=int(os.environ.get("FPH_BENCH_LANES", "2")))


def step_sharded(lib, native, w, stream):
    """N > 1: this rank's spatially compact share of every dimension in one
    fph_flood_subset call (grid built once; the shares are Morton-ordered
    cuts of the simplex centers, computed once per complex in prepare),
    NCCL all-gather back into row order, then facet completion on every
    rank."""
    import torch.distributed as dist

    from paper_2509_22432_b200.parallel import flood_sq_values_spatial

    Xd, dc = w["items"][0]
    by_dim = {0: w["vert_ids"], **dc.simp}
    vals = flood_sq_values_spatial(Xd, dc.lm, by_dim, dc.facets, dc.top, w["m"], dist, w["parts"])
    for k in range(dc.top + 1):
        dc.out[k][: vals[k].shape[0]] = vals[k]


def shard_parts(w, world):
    """Every rank computes the same spatial partition of each dimension's
    simplices (parallel.spatial_partition: Morton order of the Ritter
    centers cut into equal counts)."""
    import torch

    from paper_2509_22432_b200.parallel import simplex_centers, spatial_partition

    tri, dc = w["tri"], w["items"][0][1]
    w["vert_ids"] = torch.arange(dc.counts_full[0], dtype=torch.int32, device=dc.dev)
    w["parts"] = {k: [torch.from_numpy(p).to(dc.dev) for p in
                      spatial_partition(simplex_centers(tri.points, tri.simplices_by_dim[k]), None,
                                        world)]
                  for k in range(1, dc.top + 1)}


def run_ours(args):
    import torch

    from paper_2509_22432_b200 import _native

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1 or args.force_sharded:
        import socket

        import torch.distributed as dist

        if "RANK" not in os.environ:  # --force-sharded without torchrun: a world of one
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                              WORLD_SIZE="1", LOCAL_RANK="0")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    lib = _native.require_gpu()
    w = prepare(args.config, local, rank)
    stream = torch.cuda.current_stream().cuda_stream
    sharded = (world > 1 or args.force_sharded) and not w["batch"]
    step = step_sharded if sharded else step_single
    if sharded:
        shard_parts(w, world)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=w["dev"])  # > 126 MB L2
    for _ in range(args.warmup):
        step(lib, _native, w, stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    lib.fph_launch_count(1)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record()
            step(lib, _native, w, stream)
            ends[i].record()
        torch.cuda.synchronize()
        launches = int(lib.fph_launch_count(0))
        # the same step captured into a CUDA graph and replayed (single-call
        # steps; values checked equal to the uncaptured step's)
        graph = (graph_step(lib, _native, w, flush, args)
                 if (step is step_single and not args.no_graph) else None)
    # an extra profiled pass (CUDA events around the flooding kernels, work
    # counters) for the roofline, outside the timed steps
    stats = np.zeros(24)
    lib.fph_set_profiling(1)
    lib.fph_flood_stats(stats.ctypes.data, 1)
    for _ in range(args.steps):
        flush.zero_()
        step(lib, _native, w, stream)
    torch.cuda.synchronize()
    lib.fph_flood_stats(stats.ctypes.data, 1)
    lib.fph_set_profiling(0)
    sharded_ok = None
    if sharded:  # the gathered values must equal a single-call pass
        dc = w["items"][0][1]
        got = [t.clone() for t in dc.out]
        step_single(lib, _native, w, stream)
        torch.cuda.synchronize()
        sharded_ok = all(torch.equal(a[: c], b[: c]) for a, b, c in zip(got, dc.out, dc.counts_full))
    ms_eager = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
    # the faster of the two launch modes of the same step (a batch's eager
    # calls on two streams can beat their graph: modelnet_batch 143 vs 154 ms)
    use_graph = (bool(graph) and graph.get("values_equal_uncaptured") is True
                 and graph["ms_per_step"] < ms_eager)
    ms = graph["ms_per_step"] if use_graph else ms_eager
    n_simplices = sum(dc.n_simplices for _, dc in w["items"])
    if not sharded and world > 1:  # weak scaling: every rank its own clouds
        t = torch.tensor([float(n_simplices)], dtype=torch.float64, device=w["dev"])
        torch.distributed.all_reduce(t)
        n_simplices = int(t.item())
    if world > 1:
        t = torch.tensor([ms, ms_eager], device=w["dev"])
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, ms_eager = float(t[0].item()), float(t[1].item())
    value = n_simplices / (ms / 1e3)

    result = None
    if rank == 0:
        e2e = e2e_host(lib, _native, w, args) if world == 1 else None
        dc0 = w["items"][0][1]
        config = {"workload": args.config, "points": w["n"], "landmarks": w["nl"],
                  "grid_resolution": w["m"], "max_dim": w["max_dim"], "simplices": n_simplices,
                  "l2": "flushed (256 MB write) between timed steps"}
        if w["batch"]:
            config.update({"clouds_per_gpu": len(w["items"]), "clouds": len(w["items"]) * world,
                           "parallelism": f"whole clouds per GPU x{world}, no collective"})
        else:
            config.update({"counts": dc0.counts_full,
                           "parallelism": f"spatial simplex shards x{world}, cloud replicated"})
        result = {
            "metric": "flood-filtration simplices/s",
            "value": value,
            "unit": "simplices/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "ms_per_step_eager": ms_eager,
            "ms_per_step_graph": graph.get("ms_per_step") if graph else None,
            "launch": ("CUDA graph of the step, replayed (values equal to the eager step's)"
                       if use_graph else "eager C-ABI calls (the faster mode)"),
            "higher_is_better": True,
            "scaling": "weak" if w["batch"] else "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "numerics": "fp32 FFMA2 filter with a rigorous error bound + exact float64 refine; "
                        "values bit-identical to the reference's float64",
            "data": "synthetic: seeded generator (" + {
                "sphere_torus": "noisy sphere+torus mix", "box": "uniform box",
                "torus": "torus surface", "modelnet": "ModelNet-shaped primitive unions"}[w["kind"]]
                    + "), no dataset download",
            "config": config,
            "fps_ms": w["fps_ms"],
            "fps_scope": ("one batched launch over this GPU's clouds" if w["batch"]
                          else "one cloud"),
            "delaunay_s": w["delaunay_s"],
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if sharded_ok is not None:
            result["sharded_equals_single_gpu_values"] = sharded_ok
        if graph:
            result["cuda_graph"] = graph
        if e2e:
            result["e2e"] = e2e
        result["roofline"] = roofline(lib, stats, ms, args.steps, clocks.summary(),
                                      brute_pairs=brute_pairs(lib, _native, w, stream),
                                      config=args.config)
        result["work_per_step"] = {"fp32_pairs": stats[0] / args.steps,
                                   "candidates_staged": stats[1] / args.steps,
                                   "candidates_scanned": stats[2] / args.steps,
                                   "refined_points": stats[3] / args.steps,
                                   "f64_refine_distances": stats[4] / args.steps,
                                   "tasks": stats[5] / args.steps,
                                   "search": {"blocks_searched": stats[7] / args.steps,
                                              "block_searches": stats[15] / args.steps,
                                              "blocks_pruned": stats[8] / args.steps,
                                              "cta_team_simplices": stats[9] / args.steps,
                                              "staged_phase_a": stats[16] / args.steps,
                                              "staged_block_sampling": stats[17] / args.steps,
                                              "staged_block_exact": stats[18] / args.steps,
                                              "phase_a_pairs": stats[14] / args.steps,
                                              "warp_cycles_a_b_c_f": [stats[19 + i] / args.steps
                                                                      for i in range(4)]}}
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
            result["fps_cpu_baseline"] = fps_cpu_baseline(w)
    if world > 1 or args.force_sharded:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return result


def roofline(lib, stats, step_ms, steps, clocks, brute_pairs=None, config="sphere_torus_1m"):
    """Flooding kernel (search_kernel, algorithm 1): FP32-pipe bound.  Work =
    6 flop (three FMAs of |a|^2 - 2 a.b) per (sample point, candidate) pair
    actually evaluated, counted on the device; time = CUDA events around
    every flooding-kernel launch on its stream during the timed steps.
    `effective` rates the same time against the reference algorithm's pair
    count (every sample point x every cloud point of the Lemma-4.2 ball),
    i.e. what a brute-force kernel would have had to sustain.  DRAM traffic,
    achieved HBM GB/s and FP32-pipe utilisation of the whole step come from
    the committed ncu range capture of one real step (caches not flushed)."""
    pairs, pass_ms = stats[0], stats[6]
    sec = pass_ms * 1e-3
    achieved = 6.0 * pairs / sec / 1e12 if pass_ms > 0 else 0.0
    peak = float(lib.fph_fp32_peak_tflops())
    out = {"bound": "fp32", "kernel": "search_kernel", "achieved": achieved, "peak": peak,
           "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": None,
           "peak_source": "measured FFMA2 microbenchmark on this GPU (fph_fp32_peak_tflops, "
                          "csrc/fph_diag.cu); MEASURED_PEAKS.json has no FP32 figure",
           "kernel_ms_per_step": pass_ms / steps, "kernel_share_of_step": pass_ms / steps / step_ms}
    cap = _step_capture(config)
    if cap:
        traffic = cap["dram_bytes_per_step"]
        peaks = _peaks()
        cycles = step_ms * 1e-3 * 1.965e9 * 148 * 4  # SMSP-cycles in the step at max clock
        out.update({
            "traffic": traffic,
            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of ONE whole step from "
                            f"{cap['_path']} (ncu --replay-mode app-range, --cache-control none)",
            "algorithmic_bytes": _algorithmic_bytes(config),
            "hbm_gbs_achieved": traffic / (step_ms * 1e-3) / 1e9,
            "hbm_gbs_peak": peaks.get("hbm_gbs"),
            "hbm_frac": (traffic / (step_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]) if peaks.get("hbm_gbs") else None,
            "fp32_pipe_util": cap["sm_inst_executed_pipe_fma"] / cycles,
            "fp32_pipe_note": "sm__inst_executed_pipe_fma of the captured step / (SMSP cycles of "
                              "the event-timed step at 1965 MHz); ncu's own "
                              "sm__pipe_fma_cycles_active over the (launch-gap inflated) range: "
                              f"{cap['sm_pipe_fma_cycles_active_pct_of_range']:.1f}%",
        })
    if brute_pairs:
        out["reference_algorithm_pairs_per_step"] = brute_pairs
        out["effective_tflops_vs_reference_algorithm"] = 6.0 * brute_pairs / (sec / steps) / 1e12
    return out


def _step_capture(config):
    path = os.path.join(ROOT, "profiles", "r02", f"ncu_step_range_{config}.json")
    try:
        with open(path) as fh:
            cap = json.load(fh)
    except (OSError, ValueError):
        return None
    cap["_path"] = os.path.relpath(path, ROOT)
    return cap


def _algorithmic_bytes(config):
    """Bytes a step must move at least: read the float64 cloud once, write
    its grid-sorted copy once, read the landmarks and complex, write the
    values ("Roofline")."""
    kind, n, nl, m, max_dim = CONFIGS[config]
    dim = 2 if kind == "circle" else 3
    return 2 * n * dim * 8


def graph_step(lib, native, w, flush, args):
    """The same step captured once into a CUDA graph (device-memory calls on
    a capturing stream: grid build, every dimension's kernels on their forked
    streams, completion) and replayed: time per replay (events, L2 flushed)
    and whether the replayed values equal an uncaptured step's."""
    import torch

    try:
        ref = [dc.out[k][: dc.counts_full[k]].clone() for _, dc in w["items"]
               for k in range(dc.top + 1)]
        s = torch.cuda.Stream(device=w["dev"])
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            step_single(lib, native, w, s.cuda_stream)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        got = [dc.out[k][: dc.counts_full[k]] for _, dc in w["items"] for k in range(dc.top + 1)]
        same = all(torch.equal(a, b) for a, b in zip(ref, got))
        n = sum(dc.n_simplices for _, dc in w["items"])
        ms = float(np.mean(times))
        return {"ms_per_step": ms, "value": n / (ms / 1e3), "values_equal_uncaptured": same}
    except Exception as e:  # report, never fail the bench line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def brute_pairs(lib, native, w, stream):
    """Pairs the reference algorithm evaluates on this complex (one untimed
    brute-force pass, algorithm 0, counts them on the device)."""
    import torch

    stats = np.zeros(24)
    native.check(lib.fph_set_search(0, 0, 0))
    lib.fph_flood_stats(stats.ctypes.data, 1)
    step_single(lib, native, w, stream)
    torch.cuda.synchronize()
    lib.fph_flood_stats(stats.ctypes.data, 1)
    native.check(lib.fph_set_search(1, 0, 0))
    return float(stats[0])


def e2e_host(lib, native, w, args):
    """Same metric through the C ABI with HOST buffers: H2D of the cloud(s)
    and complex(es), the GPU pass, D2H of the values, all inside the timed
    region (pinned host memory)."""
    import torch

    top = w["max_dim"]

    def pinned(a):  # page-locked copy: the contract's "pinned host memory"
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    calls, h2d, d2h = [], 0, 0
    for X, tri in zip(w["Xs"], w["tris"]):
        Xp, lm = pinned(X), pinned(tri.points)
        counts = np.array([tri.simplices_by_dim[k].shape[0] for k in range(top + 1)], dtype=np.int64)
        simp = [None] + [pinned(tri.simplices_by_dim[k].astype(np.int32)) for k in range(1, top + 1)]
        fac = [None] + [pinned(tri.facet_links[k].astype(np.int32)) for k in range(1, top + 1)]
        outs = [pinned(np.empty(max(int(c), 1))) for c in counts]
        h2d += Xp.nbytes + lm.nbytes + sum(a.nbytes for a in simp[1:]) + sum(a.nbytes for a in fac[1:])
        d2h += int(sum(counts) * 8)
        calls.append((Xp, lm, counts, native.ptr_array(simp, None), native.ptr_array(fac, None),
                      native.ptr_array(outs, None), simp, fac, outs))
    nsimp = sum(int(c[2].sum()) for c in calls)

    def run_share(share):
        for Xp, lm, counts, sp, fp, op, *_ in share:
            native.check(lib.fph_flood_filtration(
                native.ptr(Xp), Xp.shape[0], Xp.shape[1], native.ptr(lm), lm.shape[0], top,
                native.ptr(counts), sp, fp, w["m"], 1, op, native.FPH_MEM_HOST, None))

    # a batch's clouds from two host threads (each host-memory call runs on
    # its thread's stream: one cloud's copies and grid build overlap the
    # other's search); one cloud: one call
    pool = ThreadPoolExecutor(max_workers=2) if len(calls) > 1 else None

    def run():
        if pool is None:
            run_share(calls)
        else:
            list(pool.map(run_share, [calls[0::2], calls[1::2]]))

    # warm-up: at least 3 calls and 0.5 s of them (a fresh box's first
    # process measured host-buffer calls ~25% slower until the copies had
    # run for a while: 5.1 vs 4.1 ms on configs[1])
    t_warm, n_warm = time.perf_counter(), 0
    while n_warm < 3 or time.perf_counter() - t_warm < 0.5:
        run()
        n_warm += 1
    times = []
    for _ in range(max(10, args.steps)):  # wall-clock: a median over >= 10 calls
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    sec = float(np.median(times))
    if pool is not None:
        pool.shutdown()
    return {"value": nsimp / sec, "unit": "simplices/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "ms_per_step": sec * 1e3}


def cpu_sample(w, seconds: float, threads: int):
    """Time the oracle (reference algorithm, C, all threads) on a random
    sample of the complex's top simplices (each with its faces, as the
    reference values them: one grid per top cell, filtration.py:246-253).
    The reference's cost is per top cell, so a sample of |S| of the n_top
    cells is credited with |S| / n_top of the complex's simplices (crediting
    the faces the sample happens to carry would over-count them ~2x)."""
    import oracle

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from tests._complex import sub_complex

    tri, top, m = w["tri"], w["max_dim"], w["m"]
    rng = np.random.default_rng(1)
    n_top = tri.simplices_by_dim[top].shape[0]
    sample = 4
    elapsed, done = 0.0, 0
    while True:
        rows = rng.choice(n_top, min(sample, n_top), replace=False)
        sub = sub_complex(tri.simplices_by_dim, rows, top)
        t0 = time.perf_counter()
        oracle.flood_values(w["X"], tri.points, sub, m, threads=threads, top_dim=top)
        dt = time.perf_counter() - t0
        total = sum(tri.simplices_by_dim[k].shape[0] for k in range(top + 1))
        nsimp = total * len(rows) / n_top
        if dt > 0.25 * seconds or sample >= n_top:
            return nsimp, dt, len(rows)
        sample = int(min(n_top, sample * max(2.0, 0.5 * seconds / max(dt, 1e-3))))


def cpu_baseline(w, seconds: float):
    threads = os.cpu_count() or 1
    nsimp, dt, ntop = cpu_sample(w, seconds, threads)
    return {"value": nsimp / dt, "unit": "simplices/s", "cores": threads, "kind": "port",
            "sample": f"{ntop} random top simplices (dim {w['max_dim']}) with their faces, "
                      f"{dt:.1f} s, credited {ntop}/{w['tri'].simplices_by_dim[w['max_dim']].shape[0]}"
                      f" of the complex's simplices ({nsimp:.0f})"}


def fps_cpu_baseline(w):
    """The oracle's farthest point sampling (reference geometry.py:88, C
    port, all host threads) on the same cloud and landmark count as fps_ms,
    checked index for index against the GPU's landmarks."""
    import oracle

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    idx = oracle.fps(w["X"], w["nl"], 0, threads=threads)
    dt = time.perf_counter() - t0
    per_cloud = w["fps_ms"] / len(w["Xs"])
    return {"value": dt * 1e3, "unit": "ms per cloud", "cores": threads, "kind": "port",
            "sample": f"full FPS of one cloud ({w['n']} points, {w['nl']} landmarks)",
            "gpu_ms_per_cloud": per_cloud, "speedup": dt * 1e3 / per_cloud,
            "indices_equal_gpu": bool(np.array_equal(idx, w["idx"]))}


def run_reference(args):
    world, rank, local = _dist()
    if rank != 0:
        return None
    import oracle
    from paper_2509_22432_b200.delaunay import delaunay

    kind, n, nl, m, max_dim = CONFIGS[args.config]
    X = _cloud(kind, n)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    idx = oracle.fps(X, nl, 0, threads=threads)  # reference algorithm (C port) for the landmarks
    fps_ms = (time.perf_counter() - t0) * 1e3
    tri = delaunay(X[idx])
    w = dict(X=X, tri=tri, m=m, max_dim=min(max_dim, tri.dim))
    for _ in range(args.warmup):
        cpu_sample(w, args.cpu_seconds / 4, threads)
    vals = []
    desc = ""
    for _ in range(args.steps):
        nsimp, dt, ntop = cpu_sample(w, args.cpu_seconds, threads)
        vals.append(nsimp / dt)
        desc = (f"{ntop} random top simplices + faces per step, credited {ntop}/"
                f"{tri.simplices_by_dim[w['max_dim']].shape[0]} of the complex ({nsimp:.0f} simplices)")
    value = float(np.median(vals))
    return {"impl": "reference", "metric": "flood-filtration simplices/s", "value": value,
            "unit": "simplices/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator)",
            "config": {"workload": args.config, "points": n, "landmarks": nl, "grid_resolution": m,
                       "max_dim": w["max_dim"]},
            "fps_ms": fps_ms,
            "cpu_baseline": {"value": value, "unit": "simplices/s", "cores": threads, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": "simplices/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def run_profile(args):
    import torch

    from paper_2509_22432_b200 import _native

    lib = _native.require_gpu()
    w = prepare(args.config, 0)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        step_single(lib, _native, w, stream)
    torch.cuda.synchronize()
    print("profile run done", [dc.counts_full for _, dc in w["items"]][:2])


def run_profile_range(args):
    import torch

    from paper_2509_22432_b200 import _native

    lib = _native.require_gpu()
    w = prepare(args.config, 0)
    stream = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=w["dev"])
    for _ in range(3):
        step_single(lib, _native, w, stream)
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    step_single(lib, _native, w, stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profile range done", [dc.counts_full for _, dc in w["items"]][:1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="sphere_torus_1m")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay measurement")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-GPU (shard + NCCL all-gather + completion) step even at N=1")
    ap.add_argument("--profile", action="store_true",
                    help="minimal run for ncu: setup, 1 warm-up step, 1 step, no e2e/cpu")
    ap.add_argument("--profile-range", action="store_true",
                    help="for ncu --replay-mode app-range: warm-up steps, an L2 flush, then ONE step "
                         "between cudaProfilerStart/Stop (the whole PDL-chained step as one range)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.profile:
        return run_profile(args)
    if args.profile_range:
        return run_profile_range(args)
    # stdout carries exactly one JSON line: anything libraries print there
    # (NCCL's version banner, CUDA/driver notices) goes to stderr instead
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    sys.stdout.flush()
    if res is not None:
        json_out.write(json.dumps(res) + "\n")
    json_out.flush()


if __name__ == "__main__":
    main()
