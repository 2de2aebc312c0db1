#!/usr/bin/env python
"""bench.py — RGB-D-N fwd+bwd training views/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "cfg2"): synthetic aerial city block,
~200k anchors x 10 gaussians (K=3 LoD levels, LoD bias 2), a batch of 8 views
at 1920x1080 per step, loss = L1 rgb + depth-prior L1 (Eq. 9, weight 1 at
step 0) + normal-prior L1 (weight 0.5). One step = cull, decode, project,
sort, bin, composite, loss, composite backward, projection backward, decode
backward for all 8 views, then the fused Adam over every parameter.
Targets are rendered by a "teacher" (same scene, different decoder seed and
embeddings) on the device before timing. Inputs (>> L2 per step: 8 views x
1080p x RGB/depth/normal targets + ~0.5 GB of per-view intermediates) are
larger than the 126 MB L2, so no explicit flush is needed.

  python bench.py [--gpus N --steps K --warmup W]            # CUDA path
  python bench.py --impl reference [--steps K --warmup W]    # reference CPU arm

N > 1 (torchrun, or `--gpus N` alone: bench.py then re-launches itself
under torch.distributed.run with N ranks, and fails if fewer GPUs exist):
the anchors are sharded over the ranks by the paper's Eq. 3 (i mod M,
partition.py:43-52) and every step runs dist.sharded_train_step: each rank
culls / decodes / projects its own anchors for all views, a C1 all-to-all
moves the splat records to each view's renderer rank, the reverse C1 returns
the 2D gradients, and a C2 all-reduce sums the decoder gradient. cfg2 is
weak scaling (8 views per rank per step); cfg3 (1M anchors, 16 views at
1080p) and cfg4 (2M anchors, 8 views at 3840x2160) keep the batch fixed
(strong scaling). Rank 0 prints one JSON line with the max-over-ranks
device time.

The reference arm runs the UNMODIFIED reference (oracle/_ref, installed by
oracle/build_ref.py from /root/reference/pkg) on the host cores: a bounded,
intersection-scaled sample of the same workload per step
(oracle/ref_bench.py), plus one full reference train_step at cfg1 with all
threads and with one thread.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

# Expandable segments (set before torch initialises CUDA): the per-step
# buffers vary in size with each view's intersection count, and with fixed
# segments the cache kept growing (cudaMalloc) several steps past warm-up.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "RGB-D-N fwd+bwd train views/sec at 1/2/4/8 B200 vs CPU ref; raster HBM GB/s"
CFG2_VOXEL = 1.119          # base voxel size giving ~200k anchors over 3 levels
CFG3_VOXEL = 0.503          # ~1M anchors (synthetic._fit_voxel, precomputed)
CFG4_VOXEL = 0.395          # ~2M anchors
CFG_LOD_BIAS = 2
CFG2_LOD_BIAS = CFG_LOD_BIAS


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["vsx", "reference"], default="vsx")
    ap.add_argument("--config", choices=["cfg2", "cfg1", "cfg3", "cfg4"], default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg1", action="store_true",
                    help="skip the same-config cfg1 side measurement")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU sharded step even at one rank (testing)")
    ap.add_argument("--deterministic", action="store_true",
                    help="TrainConfig.deterministic: fixed-order gradient / loss sums (a side "
                         "measurement of the mode's cost; the headline runs the default)")
    ap.add_argument("--cpu-tiles", type=int, default=40,
                    help="tiles composited per reference sample in the cpu_baseline leg")
    ap.add_argument("--ref-tiles", type=int, default=40,
                    help="tiles per --impl reference step (each of the W+K steps is one "
                         "such sample, so the arm ends within a few minutes)")
    ap.add_argument("--ref-cfg1-threads", default="all,1",
                    help="thread counts of the full reference cfg1 step in --impl reference "
                         "('all' = os.cpu_count(); empty = skip)")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ workload

CITY = {  # config -> (target anchors, base voxel, views per step, width, height, scaling)
    "cfg2": (200_000, CFG2_VOXEL, 8, 1920, 1080, "weak"),
    "cfg3": (1_000_000, CFG3_VOXEL, 16, 1920, 1080, "strong"),
    "cfg4": (2_000_000, CFG4_VOXEL, 8, 3840, 2160, "strong"),
}


def workload(config: str, world: int = 1):
    """(scene, views, config description, host images or None).

    cfg2 is weak scaling: 8 views per rank per step. cfg3 / cfg4 keep their
    batch (16 views at 1080p / 8 views at 4K) for every world size."""
    from paper_2503_23044_b200.synthetic import cfg1_scene, city_scene, city_views
    if config == "cfg1":
        scene, views, images = cfg1_scene()
        return scene, views, {"workload": "cfg1: 10,198 anchors x 10 gaussians, 4 views 128x128",
                              "anchors": scene.total_voxels, "views_per_step": 4,
                              "resolution": "128x128", "loss": "rgb"}, images
    target, voxel, nv, W, H, scaling = CITY[config]
    scene, views = city_scene(target_anchors=target, base_voxel_size=voxel, n_views=nv,
                              width=W, height=H)
    scene.lod_bias = CFG_LOD_BIAS
    if scaling == "weak" and world > 1:
        views = city_views(nv * world, W, H)
    desc = {"workload": f"{config}: synthetic aerial city block, {target // 1000}k anchors x 10 "
                        f"gaussians (K=3, LoD bias {CFG_LOD_BIAS}), {nv} views/step"
                        f"{' per GPU' if scaling == 'weak' else ''} at {W}x{H}, RGB+depth+normal"
                        " loss",
            "anchors": scene.total_voxels, "gaussians_total": scene.total_voxels * 10,
            "views_per_step": len(views), "resolution": f"{W}x{H}",
            "loss": "L1 rgb + depth-prior L1 (Eq.9) + 0.5 normal-prior L1",
            "l2_flush": "inputs > L2 (per-step working set ~GBs)"}
    return scene, views, desc, None


def config_of(args, world: int, desc: dict) -> dict:
    """The JSON `config` object, identical for the CUDA and the reference arm."""
    desc = dict(desc)
    desc["parallelism"] = (f"anchor-sharded x{world} (Eq.3 i mod M), views rendered round-robin, "
                           "C1 all-to-all + C2 decoder all-reduce (NCCL)") if world > 1 else "single"
    desc["scaling"] = CITY.get(args.config, (0, 0, 0, 0, 0, "weak"))[5]
    if getattr(args, "deterministic", False):
        desc["sums"] = "fixed-order (TrainConfig.deterministic)"
    return desc


def teacher_targets(scene, views):
    """Render RGB / depth / normal targets with a perturbed teacher on the device."""
    import torch
    from paper_2503_23044_b200 import device as D
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState
    teacher = TrainState(scene, TrainConfig(seed=7, total_steps=10, step2_start=10,
                                                step3_start=10, growth_stop=0))
    g = torch.Generator(device="cuda").manual_seed(7)
    with torch.no_grad():
        teacher.anchors.emb.add_(torch.randn(teacher.anchors.emb.shape, generator=g,
                                             device="cuda") * 0.5)
    ds = teacher.dscene
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = []
    for v in views:
        act = ds.active(v)
        dec = D.decode(teacher.params.abi(), teacher.n, act, ds.centers, teacher.anchors.emb,
                       teacher.anchors.log_scales, teacher.anchors.offsets, v, ds.lod_ref,
                       ds.max_scale, status, keep_cache=False)
        P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v,
                      status)
        R = D.raster_forward(P, D.bin_tiles(P, v.width, v.height), v)
        out.append({"rgb": R.rgb.clone(), "depth": R.depth.clone(), "valid": R.valid.clone(),
                    "normal": R.normal.clone()})
    D.check_status(status, "teacher")
    del teacher
    return out


# ------------------------------------------------------------------ clocks

class NvmlClockSampler:
    """SM clock + clock-event reasons sampled in-process (NVML) every 100 ms.

    NVML is initialised at construction (before warm-up) so its start-up cost
    never lands in the timed region; the sampling thread only runs while the
    timed steps run. Falls back to ClockSampler (nvidia-smi) if NVML fails.
    """

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu: int):
        import threading
        import pynvml
        import torch
        self.nv = pynvml
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(gpu)
        try:
            self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(p.uuid))
        except Exception:
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        self.rows: list[tuple[float, int]] = []
        self.cost: list[float] = []
        self.ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _sample(self):
        nv = self.nv
        t = time.perf_counter()
        self.rows.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                          int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
        self.cost.append(time.perf_counter() - t)

    def _run(self):
        while True:
            self._sample()
            if self.ev.wait(0.1):
                break

    def start(self):
        self.th.start()

    def stop(self) -> dict:
        self.ev.set()
        self.th.join()
        self._sample()
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, bits in self.rows for n, b in self.REASONS if bits & b})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "src": "nvml",
                "max_query_ms": round(1e3 * max(self.cost), 2)}


class _NoClocks:
    def start(self):
        pass

    def stop(self) -> dict:
        return {"src": "disabled (VSX_NO_CLOCKS=1)"}


def clock_sampler(gpu: int):
    if os.environ.get("VSX_NO_CLOCKS") == "1":
        return _NoClocks()
    try:
        return NvmlClockSampler(gpu)
    except Exception:
        return ClockSampler(gpu)


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path(tempfile.mkstemp(prefix="clocks_", suffix=".csv")[1])

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture, or None."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return int(json.loads(p.read_text())[kernel]["bytes"])
    except Exception:
        return None


def ncu_limiter(kernel: str):
    """The limiter the committed ncu capture shows for `kernel` (issue slots)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        e = json.loads(p.read_text())[kernel]
        return {"kind": "instruction issue", "ncu_issue_slots_busy": e["issue_slots_busy"],
                "source": e["source"]}
    except Exception:
        return None


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------ CPU baseline (oracle)

def reference_available() -> bool:
    from oracle.ref_bench import REF_DIR
    return (REF_DIR / "voxsplat" / "__init__.py").exists()


def reference_sampler(config: str, views, tiles: int, front_views: int):
    """oracle/ref_bench.Cfg2Sampler on the same points / views as the CUDA arm."""
    import torch
    from oracle.ref_bench import Cfg2Sampler
    from paper_2503_23044_b200.synthetic import city_points
    torch.set_num_threads(os.cpu_count() or 1)
    target, voxel, _nv, _W, _H, _ = CITY[config]
    pts = city_points(n_points=max(600_000, int(7.5 * target)), seed=0)
    return Cfg2Sampler(pts, voxel, 3, CFG_LOD_BIAS, 10, views, tiles, normal_weight=0.5,
                       front_views=front_views)


def _ref_sample_desc(s, r: dict, n: int) -> str:
    return (f"UNMODIFIED reference (oracle/_ref voxsplat, float64) on the host cores, "
            f"{n} samples of the workload: per sample the reference's rasterize_view buckets "
            f"(_blend_padded + _finalize) fwd + autograd bwd on {r['tiles']} of "
            f"{r['tiles_nonempty']} non-empty tiles of one view ({r['isect_sampled']} of "
            f"{r['isect_total']} intersections, scaled by intersections), RGB + Eq.9 depth + "
            f"normal-prior L1, + the view's transfer_gaussians/project_splats/bin_splats "
            f"({r['front_s']:.1f} s) and projection+decode autograd ({r['proj_decode_bwd_s']:.1f}"
            f" s) measured once per view at setup ({len(s.fronts)} views), + the reference Adam "
            f"over all parameters per sample ({r['adam_s']:.2f} s); step = "
            f"{len(s.views)} views + 1 Adam")


def cpu_sample(config: str, views, tiles: int) -> dict:
    """cpu_baseline of the CUDA arm: the reference on a bounded sample (one
    front-end view, 2 tile samples, ~30 s), or the oracle port if the
    reference is not installed."""
    import torch
    if config != "cfg1" and reference_available():
        t0 = time.perf_counter()
        s = reference_sampler(config, views, tiles, front_views=1)
        rs = [s.sample() for _ in range(2)]
        value = float(np.median([r["views_per_s"] for r in rs]))
        return {"value": value, "unit": "views/s", "cores": torch.get_num_threads(),
                "kind": "reference", "wall_s": time.perf_counter() - t0,
                "sample": _ref_sample_desc(s, rs[-1], len(rs))}
    return cpu_sample_port(*workload(config)[:2], tiles=2000)


def cpu_sample_port(scene, views, tiles: int, images=None) -> dict:
    """Oracle (float64 CPU port) on ONE view of the workload, time-extrapolated.

    Full cull/decode/project/bin for the view, composite fwd+bwd on `tiles`
    evenly spaced non-empty tiles, full projection+decode backward; the tile
    time is scaled by intersections(total)/intersections(sampled).
    """
    import torch
    import oracle
    torch.set_num_threads(os.cpu_count() or 1)
    n = scene.offsets_per_voxel
    w = oracle.decoder_init(n, 0, float(np.log(0.125 * scene.base_voxel_size)))
    st = oracle.OracleState.create(
        scene.flat_centers(), scene.flat_levels(), scene.lod_count, scene.lod_ref_distance,
        scene.lod_bias, scene.base_voxel_size, n, w, scene.flat("embeddings"),
        np.log(scene.flat("scales")), scene.flat("offsets"), total_steps=30000)
    v = views[0]
    img = images[0] if images is not None else \
        np.random.default_rng(0).uniform(0, 1, (v.height, v.width, 3))
    t0 = time.perf_counter()
    oracle.train_step(st, [oracle.Cam.of(v)], [img], tile_limit=tiles)
    wall = time.perf_counter() - t0
    tm = st.last_timing
    t_tiles = tm["t_tiles"] * tm["isect_total"] / max(tm["isect_sampled"], 1)
    t_view = tm["t_fixed"] + t_tiles
    return {"value": 1.0 / t_view, "unit": "views/s", "cores": torch.get_num_threads(),
            "kind": "port", "wall_s": wall,
            "sample": (f"oracle/ float64 port, 1 view of the workload: full cull/decode/project/"
                       f"bin, composite fwd+bwd on {tm['tiles_done']} of {tm['tiles_nonempty']} "
                       f"non-empty tiles ({tm['isect_sampled']} of {tm['isect_total']} "
                       f"intersections, extrapolated by intersections), RGB L1 term, "
                       f"Adam excluded; {wall:.1f}s measured")}


def reference_cfg1(spec: str) -> dict:
    """Full reference train_step at cfg1 (the CPU-runnable config) per thread count."""
    from oracle.ref_bench import cfg1_step_seconds
    out = {}
    for tok in [t.strip() for t in spec.split(",") if t.strip()]:
        n = (os.cpu_count() or 1) if tok == "all" else int(tok)
        r = cfg1_step_seconds(n)
        out[f"threads_{n}"] = {"views_per_s": r["views_per_s"], "step_s": r["seconds"],
                               "threads": n}
    return out


def run_reference(args):
    """--impl reference: the unmodified reference on the host cores (rank 0 only)."""
    import torch
    world, rank, _ = dist_env()
    if rank != 0:
        return
    world = max(world, args.gpus)     # the CUDA arm's config at the same N
    if not reference_available():
        from oracle.build_ref import build
        if not build():
            print(json.dumps({"impl": "reference", "unavailable":
                              "oracle/_ref not installed and /root/reference absent"}))
            return
    _scene, views, desc, _images = workload(args.config, world)
    config = config_of(args, world, desc)
    torch.set_num_threads(os.cpu_count() or 1)
    cores = torch.get_num_threads()
    t0 = time.perf_counter()
    if args.config == "cfg1":
        from oracle.ref_bench import cfg1_step_seconds
        runs = [cfg1_step_seconds(cores) for _ in range(max(1, min(args.steps, 3)))]
        value = float(np.median([r["views_per_s"] for r in runs]))
        sample = (f"UNMODIFIED reference train_step at cfg1 (full steps, {len(runs)} timed, no "
                  "warm-up: CPU float64)")
    else:
        s = reference_sampler(args.config, views, args.ref_tiles, front_views=2)
        rs = []
        for i in range(args.warmup + args.steps):
            r = s.sample()
            if i >= args.warmup:
                rs.append(r)
        value = float(np.median([r["views_per_s"] for r in rs]))
        sample = _ref_sample_desc(s, rs[-1], len(rs))
    wall = time.perf_counter() - t0
    cfg1 = reference_cfg1(args.ref_cfg1_threads) if args.ref_cfg1_threads else None
    ms = len(views) / value * 1e3
    line = {"metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": config["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "views/s", "cores": cores,
                             "kind": "reference", "sample": sample, "wall_s": wall},
            "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
            "cfg1_full_step": cfg1}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ CUDA arm

def raster_bytes(stage: str, isect: int, pixels: int, splats: int) -> int:
    """Algorithmic bytes per raster launch."""
    if stage == "raster_fwd":
        return isect * (4 + 52) + pixels * 48
    return isect * 56 + pixels * (32 + 28) + splats * 52


def run_vsx(args):
    import torch
    world, rank, local = dist_env()
    sharded = world > 1 or args.sharded
    if sharded:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0",
                              WORLD_SIZE="1")
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2503_23044_b200 import _lib
    from paper_2503_23044_b200.trainer import GpuTimer, TrainConfig, TrainState, train_step
    lib = _lib.load()
    scene, views, desc, images = workload(args.config, world)
    cfg2 = args.config != "cfg1"      # the city configs share cfg2's objective
    cfg = TrainConfig(total_steps=30000, batch_size=len(views), step2_start=0 if cfg2 else 30000,
                      step3_start=30000, growth_stop=0, normal_weight=0.5 if cfg2 else 0.0,
                      workers=world, deterministic=bool(getattr(args, "deterministic", False)))
    if cfg2:
        tgt = teacher_targets(scene, views)
        imgs = [t["rgb"] for t in tgt]
        priors = [(t["depth"], t["valid"]) for t in tgt]
        nprior = [(t["normal"], t["valid"]) for t in tgt]
    else:
        imgs = [torch.as_tensor(np.asarray(im, np.float32)).cuda() for im in images]
        priors = nprior = None
    state = TrainState(scene, cfg)
    if sharded:
        from paper_2503_23044_b200.dist import CudaShardBackend, sharded_train_step
        backend = CudaShardBackend(state, rank, world)

        def step(im, pr, npr, timer=None):
            backend.timer = timer
            r = sharded_train_step(backend, views, im, pr, npr)
            return dict(r, intersections=backend.isects)
    else:
        def step(im, pr, npr, timer=None):
            r = train_step(state, views, im, pr, normal_priors=npr, timer=timer)
            return {"gaussians": r.gaussians, "intersections": r.intersections, "total": r.total,
                    "rgb": r.rgb, "depth": r.depth, "normal": r.normal,
                    "live_pairs": r.live_pairs}
    clocks = clock_sampler(local)
    # warm-up runs the timed loop's exact code path (stage timer included):
    # on a fresh box the first touch of a code page or a lazily loaded kernel
    # module costs tens of ms, which must not land in the timed region
    for i in range(args.warmup):
        if i == args.warmup - 2:
            clocks.start()
        step(imgs, priors, nprior, GpuTimer())
    torch.cuda.synchronize()
    # head-room in every stream's cache pool so a view with more
    # intersections than any warm-up view does not map new device memory
    # inside the timed region
    from paper_2503_23044_b200.trainer import reserve_stream_pools
    reserve_stream_pools(1 << 30)
    if world > 1:
        dist.barrier()
    if args.warmup < 2:
        clocks.start()
    timer = GpuTimer()
    launches0 = lib.vsx_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    diag = os.environ.get("VSX_BENCH_DIAG") == "1"
    if diag:
        import gc
        gc0 = [g["collections"] for g in gc.get_stats()]
        m0 = torch.cuda.memory_stats()
    ev0.record()
    reps = []
    marks = []
    from paper_2503_23044_b200 import trainer as _trainer
    tr_marks = []
    for _ in range(args.steps):
        tr_marks.append(len(_trainer.TRACE_LOG))
        reps.append(step(imgs, priors, nprior, timer))
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append(e)
    tr_marks.append(len(_trainer.TRACE_LOG))
    ev1.record()
    torch.cuda.synchronize()
    if diag:
        m1 = torch.cuda.memory_stats()
        keys = ("num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams")
        print("diag alloc", {k: m1.get(k, 0) - m0.get(k, 0) for k in keys},
              "gc", [g["collections"] - c for g, c in zip(gc.get_stats(), gc0)],
              "reserved GB", m1["reserved_bytes.all.current"] / 1e9, file=sys.stderr)
    step_ms = [round(ev0.elapsed_time(marks[0]), 2)] + [
        round(a.elapsed_time(b), 2) for a, b in zip(marks, marks[1:])]
    if _trainer.TRACE_LOG:  # VSX_TRACE=1: host phase gaps of the slowest step
        k = int(np.argmax(step_ms))
        seg = _trainer.TRACE_LOG[tr_marks[k]:tr_marks[k + 1]]
        print("trace step", k, step_ms[k], [(b[0], round(1e3 * (b[1] - a[1]), 2))
                                           for a, b in zip(seg, seg[1:])], file=sys.stderr)
    clk = clocks.stop()
    launches = lib.vsx_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stage_ms = timer.totals_ms()
    stage_n = timer.counts()
    # roofline of the dominant single-launch compositing kernel
    isect = sum(r["intersections"] for r in reps)
    pixels = sum(v.width * v.height for v in views) * args.steps // world
    splats = sum(r["gaussians"] for r in reps)
    live_pairs = sum(r.get("live_pairs", 0) for r in reps)
    dom = max(("raster_fwd", "raster_bwd"), key=lambda k: stage_ms.get(k, 0.0))
    per_launch_bytes = raster_bytes(dom, isect, pixels, splats) / stage_n[dom]
    per_launch_s = stage_ms[dom] / 1e3 / stage_n[dom]
    peaks = measured_peaks()
    achieved = per_launch_bytes / per_launch_s / 1e9
    value = len(views) / (ms / 1e3)    # whole job: every view of the step, all ranks
    # end to end through the public API with host buffers (pinned H2D + loss D2H)
    e2e = None
    if not args.no_e2e:
        himgs = [t.cpu().pin_memory() for t in imgs]
        # masks travel as uint8 (one byte each, the kernels' type), so the copy
        # is a plain DMA with no cast on either side
        hpri = [(d.cpu().pin_memory(), v.cpu().to(torch.uint8).pin_memory())
                for d, v in priors] if priors else None
        hnrm = [(nn.cpu().pin_memory(), v.cpu().to(torch.uint8).pin_memory())
                for nn, v in nprior] if nprior else None
        h2d = sum(t.numel() * t.element_size() for t in himgs)
        if hpri:
            h2d += sum(d.numel() * 4 + v.numel() for d, v in hpri)
        if hnrm:
            h2d += sum(nn.numel() * 4 + v.numel() for nn, v in hnrm)
        prefetch = world == 1 and not args.sharded and os.environ.get("VSX_BENCH_E2E_DEVICE") != "1"
        # host-input path: its H2D staging buffers (two batches in flight when
        # prefetching) join the pools before the timed region
        if prefetch:
            from paper_2503_23044_b200.trainer import StagedInputs
            nxt = StagedInputs(views, himgs, hpri, hnrm)
            for _ in range(3):
                cur, nxt = nxt, StagedInputs(views, himgs, hpri, hnrm)
                step(cur, None, None)
            del nxt
        else:
            for _ in range(2):
                step(himgs, hpri, hnrm)
        reserve_stream_pools(1 << 30)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if os.environ.get("VSX_BENCH_DIAG") == "1":
            em0 = torch.cuda.memory_stats()
        if prefetch:
            # double-buffered input pipeline: step k+1's H2D copies are issued
            # (trainer.StagedInputs) before step k runs, so they overlap its
            # compute; every step's inputs are still copied inside the region
            from paper_2503_23044_b200.trainer import StagedInputs
            e0.record()
            nxt = StagedInputs(views, himgs, hpri, hnrm)
            for k in range(args.steps):
                cur = nxt
                if k + 1 < args.steps:
                    nxt = StagedInputs(views, himgs, hpri, hnrm)
                step(cur, None, None)
            e1.record()
        else:
            e0.record()
            if os.environ.get("VSX_BENCH_E2E_DEVICE") == "1":   # diagnostic: device inputs
                for _ in range(args.steps):
                    step(imgs, priors, nprior)
            else:
                for _ in range(args.steps):
                    step(himgs, hpri, hnrm)
            e1.record()
        torch.cuda.synchronize()
        if os.environ.get("VSX_BENCH_DIAG") == "1":
            em1 = torch.cuda.memory_stats()
            print("diag e2e alloc", {k: em1.get(k, 0) - em0.get(k, 0) for k in (
                "num_device_alloc", "num_device_free", "num_alloc_retries",
                "num_sync_all_streams")}, file=sys.stderr)
        ems = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": len(views) / (ems / 1e3), "unit": "views/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 * 4 + 8,
               "input_pipeline": "next step's H2D issued before the current step (StagedInputs)"
               if prefetch else "each step's H2D issued at its start"}
    cfg1 = None
    if rank == 0 and world == 1 and args.config != "cfg1" and not args.no_cfg1:
        cfg1 = cfg1_gpu(max(args.steps, 10))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.config, views, args.cpu_tiles)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    config = config_of(args, world, desc)
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": config["scaling"], "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": config,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": ncu_traffic(dom),
                     "peak_src": peaks["src"],
                     "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_s * 1e3,
                     # the compositor is issue-bound, not HBM-bound: composited
                     # (pixel, splat) pairs per second of the dominant kernel
                     "live_pairs_per_launch": live_pairs / max(stage_n[dom], 1),
                     "pairs_per_s": live_pairs / max(stage_n[dom], 1) / per_launch_s,
                     "limiter": ncu_limiter(dom)},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk,
        "stages_ms_per_step": {k: v / args.steps for k, v in stage_ms.items()},
        "step_ms": step_ms,
        "per_step": {"gaussians": reps[-1]["gaussians"],
                     "intersections": reps[-1]["intersections"],
                     "live_pairs": reps[-1].get("live_pairs"),
                     "loss_total": reps[-1]["total"], "loss_rgb": reps[-1]["rgb"],
                     "loss_depth": reps[-1]["depth"], "loss_normal": reps[-1]["normal"]},
        # same-config side measurement against the reference arm's cfg1_full_step
        "cfg1_full_step": cfg1,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def cfg1_gpu(steps: int) -> dict:
    """cfg1 (the reference's CPU-runnable config) through train_step on the
    device: views/s over `steps` timed steps after 3 warm-ups (CUDA events)."""
    import torch
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
    scene, views, _desc, images = workload("cfg1")
    st = TrainState(scene, TrainConfig(total_steps=30000, batch_size=4, step2_start=30000,
                                       step3_start=30000, growth_stop=0))
    imgs = [torch.as_tensor(np.asarray(im, np.float32)).cuda() for im in images]
    for _ in range(3):
        train_step(st, views, imgs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        train_step(st, views, imgs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"views_per_s": len(views) / (ms / 1e3), "ms_per_step": ms, "steps": steps,
            "workload": "cfg1: 10,198 anchors x 10, 4 views 128x128, RGB L1 + Adam"}


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: N ranks via torch.distributed.run."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) are visible",
              file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
           str(_free_port()), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus:
        print(f"bench.py: WORLD_SIZE={env_world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and env_world is None:
        sys.exit(relaunch(args.gpus))
    else:
        run_vsx(args)


if __name__ == "__main__":
    main()
