#!/usr/bin/env python3
"""bench.py — recycled path-segments/s per render+gradient iteration (BASELINE.json metric).

Default workload (BASELINE.json configs[1]): synthetic
128^3 single-type Gaussian cloud (peak beta 20, sigma 0.22, albedo 0.99, HG g = 0.85),
sun at zenith, 9 cameras at 128x128, 1e8 paths traced at seed 7 and sorted by B.
One timed step = one recycled Algorithm-2 iteration on the device: K3 prep -> K4
recycled forward -> image allreduce -> loss/residual -> K5 gradient -> gradient
allreduce -> K6 ADAM.  Segments = sum of B over the store (dead final segments
included).  The store (~60 GB at 1e8 paths) is far larger than L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config a|b|c|d] [--paths N]
  python bench.py --impl reference ...   (the reference's CPU path, oracle/_ref)
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2110_00085_b200 import scene as S  # noqa: E402

CONFIGS = {
    # name: (grid n, rows, species, default paths, description)
    "a": dict(n=32, rows=64, two=False, paths=1_000_000,
              desc="synthetic 32^3 single-type cloud, HG g=0.85, 9 cameras 64x64, 1e6 paths"),
    "b": dict(n=128, rows=128, two=False, paths=100_000_000,
              desc="synthetic 128^3 single-type cloud, 9 cameras 128x128, 1e8 paths, sort+recycle render+gradient"),
    "c": dict(n=128, rows=128, two=True, paths=100_000_000,
              desc="2-species 128^3 cloud (HG 0.85 + Rayleigh), 9 cameras 128x128, 1e8 paths, per-type gradients"),
    "d": dict(n=0, rows=256, two=False, paths=10_000_000,
              desc="reflectometry: Phong sphere + 14 diffuse spheres in a Phong box, 16 views 256x256, 1e7 paths"),
    # (e): 1e9 paths over the job, at most 1.25e8 per GPU (the store is ~1.2 KB/path, so
    # 1e9 needs 8 GPUs of 180 GB); recycled iterations timed as in (b), resampling every
    # N_r = 30 iterations reported amortised
    "e": dict(n=256, rows=128, two=False, paths=1_000_000_000, per_gpu_cap=125_000_000,
              desc="tomography of a 256^3 cloud, 9 cameras 128x128, 1e9 paths over the job "
                   "(<= 1.25e8 per GPU), resampled every 30 iterations"),
}
CPU_SAMPLE_PATHS = {"a": 200_000, "b": 60_000, "c": 50_000, "d": 1_000_000, "e": 30_000}
RECYCLE_PERIOD = 30  # N_r for the amortised rate


def make_scene(cfg):
    c = CONFIGS[cfg]
    if cfg == "d":
        return S.reflectometry_scene(c["rows"], c["rows"], 16)
    return S.cloud_scene(c["n"], c["rows"], c["rows"], two_species=c["two"])


def t_params(scene):
    """Recycle point beta_t = beta_ref (1 + 0.01 (v mod 5))."""
    if scene.unknown_species() >= 0:
        return S.ParamSet(S.recycle_point(scene.species[scene.unknown_species()].extinction))
    return S.ParamSet(None, 0.55, 38.0)


def max_bounces(cfg):
    return 500


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.stop = device, [], threading.Event()

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(cfg):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel per launch, from
    the committed ncu capture of the same config (profiles/ncu_traffic.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return t[cfg]["dram_bytes_per_launch"]
    except Exception:
        return None


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        if torch.cuda.device_count() < world:  # every rank exits: no rank left waiting in a collective
            raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, {torch.cuda.device_count()} visible")
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control plane only; data path is our NCCL comm
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def reduce_max(pg, x):
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(pg, x):
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t)
    return float(t.item())


# ------------------------------------------------------------------ our arm
def run_ours(args):
    from paper_2110_00085_b200.gpu import Context, EvalOptions, RenderOptions
    world, rank, local, pg = dist_setup(args.gpus)
    if world > 1:
        nid = [Context.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(nid, src=0)
        ctx = Context(local, rank, world, nid[0])
    else:
        ctx = Context(local)
    cfg = args.config
    scene = make_scene(cfg)
    n_paths = int(args.paths or CONFIGS[cfg]["paths"])
    if args.paths is None and "per_gpu_cap" in CONFIGS[cfg]:
        n_paths = min(n_paths, CONFIGS[cfg]["per_gpu_cap"] * world)
    if args.mode is not None:
        ctx.set_option("mode", args.mode)
    if CONFIGS[cfg]["two"]:
        ctx.set_option("per_species", 1)  # config (c): per-type gradients every iteration
    if args.spread is not None:
        ctx.set_option("spread", args.spread)
    if args.packet is not None:
        ctx.set_option("packet", args.packet)
    if args.grad_copies is not None:
        ctx.set_option("grad_copies", args.grad_copies)
    ctx.upload(scene)
    tp = t_params(scene)
    # warm-up resample at the full store size (another seed): loads every kernel module (CUDA
    # lazy loading), sizes the context's scratch and maps the store's memory once, so the
    # timed resample below is a steady-state one of the loop (inverse.cpp:175-204 frees the
    # previous generation and traces the next every recycle_period iterations); first-touch
    # allocations otherwise vary by 10x with what ran on the box before
    warm = ctx.render(scene, RenderOptions(n_paths=n_paths, seed=1, keep_paths=True,
                                           max_bounces=max_bounces(cfg), images=False)).store
    ctx.sort_by_size(warm)
    ctx.opt_init(tp, np.zeros(scene.pixel_count), alpha=1e-3)
    ctx.opt_step(warm)
    warm.free()
    # the resample phase of the loop (inverse.cpp:175-204): trace (K1) + sort (K2); the
    # resample iteration's forward is the recycled one at the sampling point
    barrier(pg)
    t0 = time.time()
    rr = ctx.render(scene, RenderOptions(n_paths=n_paths, seed=7, keep_paths=True,
                                         max_bounces=max_bounces(cfg), images=False))
    t1 = time.time()
    store = rr.store
    if not args.no_sort:
        ctx.sort_by_size(store)
    t2 = time.time()
    info = store.info()
    stats = ctx.store_stats(store)  # global (allreduced)
    seg_global = reduce_sum(pg, info["segments"])
    vert_global = reduce_sum(pg, info["vertices"])
    # the first forward over a fresh store (here the reference image F_ref at the sampling
    # point, the resample iteration's forward) also builds the Morton vertex table and the
    # event-geometry cache: its time beyond a steady forward is charged to the resample phase
    t3 = time.perf_counter()
    gt = 0.9 * ctx.recycled_render(scene, store, None)  # synthetic measurement: residual = F_t - 0.9 F_ref
    first_fwd_ms = reduce_max(pg, (time.perf_counter() - t3) * 1e3)
    ctx.opt_init(tp, gt, alpha=1e-3)
    for _ in range(args.warmup):
        ctx.opt_step(store)
    # ---- timed region: exactly K recycled iterations
    barrier(pg)
    launches0 = ctx.kernel_launches()
    fwd_ms = grad_ms = fwd_pp_ms = grad_pp_ms = 0.0
    with ClockSampler(local) as clk:
        ctx.timer_start()
        for _ in range(args.steps):
            ctx.opt_step(store)
            tm = ctx.last_timings()
            fwd_ms += tm["forward"]
            grad_ms += tm["gradient"]
            fwd_pp_ms += tm["forward_per_path"]
            grad_pp_ms += tm["gradient_per_path"]
        ms = ctx.timer_stop()
    barrier(pg)
    launches = ctx.kernel_launches() - launches0
    ms_max = reduce_max(pg, ms)
    trace_s, sort_s = reduce_max(pg, t1 - t0), reduce_max(pg, t2 - t1)  # resample phase (K1 + K2)
    ms_per_step = ms_max / args.steps
    value = seg_global / (ms_per_step / 1e3)
    fwd_ms /= args.steps
    grad_ms /= args.steps
    fwd_pp_ms /= args.steps
    grad_pp_ms /= args.steps
    # ---- roofline: algorithmic bytes per pass = 8 W_live + 64 V + 16 E
    W_live = stats["live_path_spans"] + stats["le_spans"]
    E = stats["events"]
    bytes_pass = 8.0 * W_live + 64.0 * vert_global + 16.0 * E
    bytes_iter = 2.0 * bytes_pass
    peak, peak_kind = measured_peak()
    # Dominant kernel (launch list: profiles/r12_kernels_1e8.md): K5b, the LE-ray gradient
    # scatter.  Its event-timed duration is the gradient phase minus K5a (+ the padded
    # fold), and its algorithmic bytes are the §8(d) per-unit figures over the units it
    # processes: 8 B per LE span incidence, 16 B per event, 64 B per vertex.
    k5b_ms = grad_ms - grad_pp_ms
    k4b_ms = fwd_ms - fwd_pp_ms
    k5b_bytes = (8.0 * stats["le_spans"] + 16.0 * E + 64.0 * vert_global) / world
    achieved = k5b_bytes / (k5b_ms / 1e3) / 1e9
    # scenes without a medium run K5b over the compact event list
    k5b_name = "k_le_gradient_ms<3> (K5b)" if scene.species else "k_evc_gradient (K5b', event list)"
    roofline = {"kernel": k5b_name, "bound": "hbm", "achieved": round(achieved, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": load_traffic(cfg), "bytes_per_launch": k5b_bytes,
                "launch_ms": round(k5b_ms, 3), "forward_ms": round(fwd_ms, 3),
                "gradient_ms": round(grad_ms, 3), "k_prefix_ms": round(fwd_pp_ms, 3),
                "k_le_forward_ms": round(k4b_ms, 3), "k_le_gradient_ms": round(k5b_ms, 3),
                "k_path_gradient_ms": round(grad_pp_ms, 3),
                "iteration_roofline_seg_per_s": seg_global / (bytes_iter / (peak * 1e9) / world),
                "iteration_frac": round(value / (seg_global / (bytes_iter / (peak * 1e9) / world)), 4)}
    # ---- e2e through the reference-facing API with host buffers
    e2e = None
    if not args.no_e2e:
        Fh = gt / 0.9
        h2d = d2h = 0
        ctx.timer_start()
        t_e2e = time.perf_counter()
        for _ in range(max(1, args.steps)):
            f = ctx.evaluate_store(scene, store, tp, EvalOptions())  # recycled_render
            res = f.images - gt
            g = ctx.evaluate_store(scene, store, tp, EvalOptions(want_grad=True, pixel_weights=res))
            _ = g.grad_beta
        e2e_ms = ctx.timer_stop() / max(1, args.steps)
        e2e_wall = (time.perf_counter() - t_e2e) / max(1, args.steps) * 1e3
        vb = 8 * scene.voxel_count
        h2d = 2 * vb + 8 * scene.pixel_count
        d2h = 2 * 8 * scene.pixel_count + (vb if scene.unknown_species() >= 0 else 16)
        e2e_ms = reduce_max(pg, max(e2e_ms, e2e_wall))
        e2e = {"value": seg_global / (e2e_ms / 1e3), "unit": "path-segments/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
               "api": "recycled_render + grad_forward (prc_gpu_evaluate x2, host buffers)"}
        del Fh
    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, scene, args.cpu_paths)
    if rank == 0:
        line = {
            "metric": "recycled path-segments/sec per render+gradient iteration",
            "value": value, "unit": "path-segments/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 geometry / f32 fields",
            "data": "synthetic (SURVEY §8(d) generator; no datasets)",
            "config": {"workload": CONFIGS[cfg]["desc"], "config": cfg, "paths": n_paths,
                       "segments": int(seg_global), "vertices": int(vert_global),
                       "events": int(E), "live_span_incidences": int(W_live),
                       "l2": "store >> L2 (126 MB), no flush needed",
                       "trace_s": round(trace_s, 4), "sort_s": round(sort_s, 4),
                       "store_setup_ms": round(max(0.0, first_fwd_ms - fwd_ms), 3),
                       "recycle_period": RECYCLE_PERIOD,
                       "amortized_seg_per_s": seg_global / (
                           ms_per_step / 1e3 + (trace_s + sort_s + max(0.0, first_fwd_ms - fwd_ms) / 1e3)
                           / RECYCLE_PERIOD),
                       "sorted_by_B": not args.no_sort,
                       "mode": "per_path" if args.mode == 1 else "wavefront",
                       "spread": args.spread, "packet": args.packet,
                       "parallelism": f"paths sharded over {world} GPU(s), NCCL allreduce"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def cpu_baseline(cfg, scene, n_cpu=None):
    """The reference's own CPU path (oracle/_ref) on the host cores, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    cores = os.cpu_count() or 1
    n = int(n_cpu or CPU_SAMPLE_PATHS[cfg])
    try:
        ref = pyoracle.Reference()
        kind = "reference"
    except Exception:
        ref, kind = None, "port"
    tp = t_params(scene)
    if ref is not None:
        st = ref.time_iteration(scene, None, tp, n, 7, cores, reps=3, warmup=1)
        secs = st["forward_s"] + st["grad_s"]
        out = {"value": st["segments"] / secs, "unit": "path-segments/s", "cores": cores,
               "kind": kind, "sample": f"{n} paths of the same workload, traced then sorted; "
               f"mean of 3 timed recycled_render + grad_forward iterations after 1 warm-up "
               f"({secs:.2f} s each, {cores} threads)",
               "forward_s": st["forward_s"], "grad_s": st["grad_s"]}
        if cores > 1:  # also the single-worker rate, on a smaller sample
            n1 = max(1000, n // 8)
            s1 = ref.time_iteration(scene, None, tp, n1, 7, 1, reps=1, warmup=0)
            out["value_1thread"] = s1["segments"] / (s1["forward_s"] + s1["grad_s"])
            out["sample_1thread"] = f"{n1} paths, 1 timed iteration, 1 thread"
        return out
    port = pyoracle.Port()
    _, _, store = port.render(scene, n, 7)
    store.sort_by_size()
    t = time.perf_counter()
    port.evaluate(scene, store, tp)
    w = np.ones(scene.pixel_count)
    port.evaluate(scene, store, tp, 3, w)
    secs = time.perf_counter() - t
    return {"value": store.stats()["segments"] / secs, "unit": "path-segments/s", "cores": 1,
            "kind": "port", "sample": f"{n} paths, oracle port single-threaded"}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    scene = make_scene(cfg)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    cores = os.cpu_count() or 1
    n = int(args.cpu_paths or CPU_SAMPLE_PATHS[cfg])
    try:
        ref = pyoracle.Reference()
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    tp = t_params(scene)
    st = ref.time_iteration(scene, None, tp, n, 7, cores, reps=max(1, args.steps),
                            warmup=max(0, args.warmup))
    secs = st["forward_s"] + st["grad_s"]
    value = st["segments"] / secs
    line = {"impl": "reference", "metric": "recycled path-segments/sec per render+gradient iteration",
            "value": value, "unit": "path-segments/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[cfg]["desc"], "config": cfg,
                       "sample_paths": n, "segments": int(st["segments"])},
            "cpu_baseline": {"value": value, "unit": "path-segments/s", "cores": cores,
                             "kind": "reference",
                             "sample": f"{n} paths of the same workload per step "
                                       f"(recycled_render + grad_forward, {cores} threads)"},
            "e2e": {"value": value, "unit": "path-segments/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="b", choices=list(CONFIGS))
    ap.add_argument("--paths", type=float, default=None)
    ap.add_argument("--cpu-paths", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sort", action="store_true", help="evaluate the unsorted (path-major) store")
    ap.add_argument("--mode", type=int, default=None, help="0 wavefront (default), 1 fused per-path")
    ap.add_argument("--spread", type=int, default=None, help="K5b lane spreading factor")
    ap.add_argument("--packet", type=int, default=None, help="K5b rays per thread in lockstep")
    ap.add_argument("--grad-copies", type=int, default=None, help="max copies of the padded gradient K5b reduces into")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}")
    if world_env is None and args.gpus > 1 and args.impl == "ours":
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
