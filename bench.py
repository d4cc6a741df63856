#!/usr/bin/env python
"""bench.py — belief updates/sec of the FP64 Algorithm-1 step on B200.

Metric (BASELINE.json): belief updates per second (Hz) — step() calls per
second — at 1024x1024x72 (configs[1], the single-GPU headline), with the HBM
GB/s of the fused step kernel against the measured peak.

One "step" is gridloc::step (belief_tensor.cpp:396-498) on the resident FP64
tensor, driven by the reference's own benchmark stream (cmd_bench,
gridloc_main.cpp:207-233: u = (res, 0, 0), main kernels, every step).

  value  : steps/s with the tensor resident in HBM (async gl_step_async,
           device time between CUDA events on the library stream, max over
           ranks); the tensor (604 MB) exceeds L2 (126 MB), so every step
           streams it from HBM.
  e2e    : the same metric through the synchronous C-ABI call a user makes
           (gl_step: host motion table -> device in the launch, status
           read back to the host every step), wall clock.
  roofline: algorithmic bytes per launch (2*8*W*H*C + W*H + 8*W*H) / the
           fused kernel's average CUDA-event duration over the timed region.
  cpu_baseline: the reference itself (oracle/_ref, compiled from the
           reference sources) on this host's cores, bounded sample.

--impl reference runs the reference's CPU implementation of the same path
(oracle/_ref; rank 0 only under torchrun) and prints the same line; it never
maps the product library (checked through /proc/self/maps).

--gpus N > 1 re-execs itself under torch.distributed.run (one rank per GPU)
unless already launched that way, and by default runs configs[3]: ONE
4096^2x360 belief theta-slab sharded across the N GPUs (strong scaling; halo
planes read over peer memory inside the step kernel, an 8-byte NCCL MAX
all-reduce per step). --config c2 with N > 1 runs independent replicas.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(W=1024, H=1024, C=72, workload="1024x1024x72 floor-plan, odometry+map correction, 1 B200 "
                                              "(BASELINE configs[1]); cmd_bench translation stream u=(res,0,0)"),
    "c1": dict(W=256, H=256, C=36, workload="256x256x36 floor-plan, odometry+map only (BASELINE configs[0])"),
    "c3": dict(W=1024, H=1024, C=72, lidar=16,
               workload="1024x1024x72 floor-plan with a LIDAR observation (belief_map -> Floyd-Steinberg budget 512 "
                        "-> likelihood update) every 16 steps (BASELINE configs[2]; cmd_bench cadence, "
                        "gridloc_main.cpp:226-244)"),
    "c5r": dict(W=512, H=512, C=72, workload="512x512x72 floor-plan (BASELINE configs[4], one robot)"),
    "c4s": dict(W=2048, H=2048, C=360, workload="2048x2048x360 floor-plan (config-4 angular width, 1/4 area)"),
    "c5": dict(W=512, H=512, C=72, batch=64, workload="batch of 64 independent robots/maps at 512x512x72 "
                                                      "(BASELINE configs[4])"),
    "c4": dict(W=4096, H=4096, C=360, workload="4096x4096x360 floor-plan, theta-slab sharded across the N GPUs "
                                              "(BASELINE configs[3]; 2 x 48.3 GB ping-pong in HBM at N = 1)"),
}
METRIC = "belief updates/sec (Hz) at 1024^2x72"  # the headline (configs[1])


def metric_for(W, H, C, lidar=0):
    if lidar:
        return f"belief updates/sec (Hz) at {W}^2x{C} with a LIDAR observation every {lidar} steps"
    return f"belief updates/sec (Hz) at {W}^2x{C}" if W == H else f"belief updates/sec (Hz) at {W}x{H}x{C}"
HBM_FALLBACK = 6650.0


def config_for(cfg):
    """The workload description both arms print (identical dicts, so the
    driver's same-config check compares like with like)."""
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    out = {"workload": cfg["workload"], "W": W, "H": H, "channels": C,
           "l2": f"inputs larger than L2: the FP64 belief ({8 * W * H * C / 1e6:.0f} MB) exceeds the 126 MB L2, "
                 "so every step streams it from HBM (no flush needed)"
           if 8 * W * H * C > 126e6 else "belief fits L2 (latency-bound small config; no flush)"}
    if cfg.get("lidar"):
        out["observe_every"] = cfg["lidar"]
        out["sample_budget"] = 512
    if cfg.get("batch"):
        out["robots_per_gpu"] = cfg["batch"]
    return out


def algo_bytes(W, H, C):
    """read + write the FP64 belief, the uint8 occupancy and
    the k-invariant FP64 activation inverse plane (isotropic kernels)."""
    return 2 * 8 * W * H * C + W * H + 8 * W * H


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def ncu_traffic(cfg_key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the fused
    kernel from the committed ncu --set full capture (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg_key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sync_boost", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
               0x100: "hw_power_brake_slowdown", 0x200: "display_clock"}

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, name in self.REASONS.items():
                if bits & b:
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(impl):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if impl == "ours":
            import torch
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def dist_max(x, world, impl):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) if impl == "ours" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def make_map_bytes(W, H):
    from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm
    return write_pgm(make_floorplan(W, H, seed=0))


# ---------------------------------------------------------------- CPU legs
def reference_engine(pgm, C, threads=0):
    import oracle
    if not oracle.ref_available():
        return None, None
    ref = oracle.Ref()
    rm = oracle.RefMap(ref, pgm=pgm)
    eng = oracle.RefEngine(ref, rm, C, threads=threads, rot_slot=False)
    return eng, rm


def lidar_scan(W, H):
    """A synthetic 24-beam, 8 m scan from the free cell nearest the centre
    (the cmd_bench scan comes from the centre, gridloc_main.cpp:224-238)."""
    import numpy as np
    from paper_1910_00572_b200.floorplan import make_floorplan, simple_scan
    occ = make_floorplan(W, H, seed=0)
    js, is_ = np.nonzero(occ == 0)
    q = int(np.argmin((is_ - W / 2) ** 2 + (js - H / 2) ** 2))
    return simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.0)


def reference_lidar_loop(eng, scan, n_steps, every, budget_s, deadline=None):
    """The reference's cmd_bench loop: step(); every `every` steps (s % every
    == 0) dither_samples(belief_map()) + observation_update()."""
    import oracle
    a, r = scan
    n = 0
    t0 = time.perf_counter()
    while n < n_steps and time.perf_counter() - t0 < budget_s:
        eng.step(0.1, 0.0, 0.0)
        if n % every == 0:
            cells, _ = oracle.ref_dither(eng.ref, eng.belief_map(), 512)
            eng.observation_update(cells, a, r, 8.0)
        n += 1
    return n, time.perf_counter() - t0


def cpu_model():
    """The host CPU model (lscpu 'Model name'), for the cpu_baseline line."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def product_not_mapped():
    """The reference arm must not map the product library."""
    try:
        maps = open("/proc/self/maps").read()
    except Exception:
        return True
    return "libgridloc_b200" not in maps


def _time_ref_steps(eng, n_max, budget_s):
    """Per-step wall times of the reference step() (u = (res, 0, 0))."""
    times = []
    t_all = time.perf_counter()
    while len(times) < n_max and time.perf_counter() - t_all < budget_s:
        t0 = time.perf_counter()
        rc = eng.step(0.1, 0.0, 0.0)
        times.append(time.perf_counter() - t0)
        if rc:
            break
    return times


def _step_stats(times):
    ts = sorted(times)
    p99 = ts[min(len(ts) - 1, int(math.ceil(0.99 * len(ts))) - 1)]
    return {"mean_ms": 1e3 * sum(ts) / len(ts), "median_ms": 1e3 * statistics.median(ts), "p99_ms": 1e3 * p99}


def cpu_baseline(pgm, cfg, budget_s=12.0, max_steps=200, one_thread_budget_s=6.0):
    """The reference's step() (oracle/_ref, compiled from the reference's own
    sources) on all host cores, bounded sample; plus a 1-thread sample
    (ThreadPool(0) and 1 thread, mean / median / p99)."""
    eng, _ = reference_engine(pgm, cfg["C"])
    if eng is None:
        return None
    eng.step(0.1, 0.0, 0.0)  # first step allocates scratch (excluded, like §6)
    model = cpu_model()
    if cfg.get("lidar"):
        n, dt = reference_lidar_loop(eng, lidar_scan(cfg["W"], cfg["H"]), max_steps, cfg["lidar"], budget_s)
        return {"value": n / dt, "unit": "Hz", "cores": eng.threads, "kind": "reference", "cpu_model": model,
                "sample": f"{n} reference step() calls with an observation every {cfg['lidar']} on "
                          f"{cfg['W']}x{cfg['H']}x{cfg['C']}, ThreadPool({eng.threads}), {dt:.1f} s"}
    times = _time_ref_steps(eng, max_steps, budget_s)
    dt = sum(times)
    out = {"value": len(times) / dt, "unit": "Hz", "cores": eng.threads, "kind": "reference", "cpu_model": model,
           "sample": f"{len(times)} reference step() calls on {cfg['W']}x{cfg['H']}x{cfg['C']} after 1 warm-up "
                     f"step, ThreadPool({eng.threads}), {dt:.1f} s"}
    out.update(_step_stats(times))
    del eng
    if one_thread_budget_s > 0:
        eng1, _ = reference_engine(pgm, cfg["C"], threads=1)
        eng1.step(0.1, 0.0, 0.0)
        t1 = _time_ref_steps(eng1, max_steps, one_thread_budget_s)
        out["one_thread"] = dict(value=len(t1) / sum(t1), unit="Hz", cores=1, steps=len(t1), **_step_stats(t1))
    return out


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    pgm = make_map_bytes(cfg["W"], cfg["H"])
    if cfg["W"] * cfg["H"] * cfg["C"] * 8 * 5 > 40e9:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the reference CPU step needs 5 tensor-sized FP64 buffers "
                          f"({cfg['W'] * cfg['H'] * cfg['C'] * 40 / 1e9:.0f} GB) for {cfg['W']}x{cfg['H']}x{cfg['C']}"}))
        return 0
    eng, _ = reference_engine(pgm, cfg["C"])
    if eng is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return 0
    if not product_not_mapped():
        raise SystemExit("reference arm: libgridloc_b200.so is mapped into this process")
    for _ in range(max(1, args.warmup)):
        eng.step(0.1, 0.0, 0.0)
    budget = args.ref_budget_s
    stats = {}
    if cfg.get("lidar"):
        n, dt = reference_lidar_loop(eng, lidar_scan(cfg["W"], cfg["H"]), args.steps, cfg["lidar"], budget)
    else:
        times = _time_ref_steps(eng, args.steps, budget)
        n, dt = len(times), sum(times)
        stats = _step_stats(times)
    assert product_not_mapped(), "reference arm mapped the product library"
    hz = n / dt
    line = {
        "impl": "reference", "metric": metric_for(cfg["W"], cfg["H"], cfg["C"], cfg.get("lidar", 0)), "value": hz,
        "unit": "Hz", "n_gpus": world, "steps": n,
        "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(n, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": f"ThreadPool({eng.threads}) host threads",
        "cpu_baseline": dict({"value": hz, "unit": "Hz", "cores": eng.threads, "kind": "reference",
                              "cpu_model": cpu_model(), "product_library_mapped": False,
                              "sample": f"{n} reference step() calls after {args.warmup} warm-up, {dt:.1f} s "
                                        f"(capped at {budget:.0f} s)"}, **stats),
        "e2e": {"value": hz, "unit": "Hz", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_reference_scaled(args, cfg, world, rank):
    """Reference arm for configs[3] (4096^2x360): the reference cannot hold
    the belief on a host (~242 GB), so each step is the reference step() at
    1024^2 with the same Theta = 360 on all host threads, and the Hz is
    scaled by the state ratio (16x) — the bounded sample of the workload,
    labelled as such."""
    if rank != 0:
        return 0
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    pgm = make_map_bytes(1024, 1024)
    eng, _ = reference_engine(pgm, C)
    if eng is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return 0
    if not product_not_mapped():
        raise SystemExit("reference arm: libgridloc_b200.so is mapped into this process")
    for _ in range(max(1, min(args.warmup, 3))):
        eng.step(0.1, 0.0, 0.0)
    times = _time_ref_steps(eng, args.steps, args.ref_budget_s)
    n, dt = len(times), sum(times)
    ratio = (1024 * 1024 * C) / (W * H * C)
    hz = n / dt * ratio
    line = {
        "impl": "reference", "metric": metric_for(W, H, C), "value": hz, "unit": "Hz", "n_gpus": world,
        "steps": n, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / hz,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": f"ThreadPool({eng.threads}) host threads",
        "cpu_baseline": dict({"value": hz, "unit": "Hz", "cores": eng.threads, "kind": "reference",
                              "cpu_model": cpu_model(), "product_library_mapped": False,
                              "scaled_from": f"1024x1024x{C}",
                              "sample": f"{n} reference step() calls at 1024x1024x{C} after warm-up, {dt:.1f} s; "
                                        f"Hz x {ratio:.4f} (state ratio): the reference cannot hold {W}x{H}x{C} "
                                        f"({W * H * C * 40 / 1e9:.0f} GB)"}, **_step_stats(times)),
        "e2e": {"value": hz, "unit": "Hz", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    assert product_not_mapped(), "reference arm mapped the product library"
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------- ours
def measure_extras(g, ctx, m, ks, act, t, cfg, args):
    """Secondary numbers on the same engine (not the headline):
    * trace_mix_hz: a recorded Localizer trace (reference simulator +
      trigger, tests/golden/trace_*.npy) — ~80% rotation-only steps (r = 0
      kernels), same algorithmic bytes per step;
    * lidar: config 3's observation cycle (belief_map -> Floyd-Steinberg
      (budget 512) -> likelihood update) latency, and the step rate with one
      observation every 16 steps (the cmd_bench cadence, gridloc_main.cpp:236).
    """
    import numpy as np
    from paper_1910_00572_b200.floorplan import make_floorplan, simple_scan
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    out = {}
    path = os.path.join(ROOT, "tests", "golden", f"trace_{W}x{C}.npy")
    if os.path.exists(path):
        tr = np.load(path)
        rk = g.build_kernels(g.MotionNoise(1e-4, 1e-4, 0.012), C, m.resolution(), 2.0 * math.pi / C)
        ract = g.make_activation(m, rk, C, ctx)
        n = min(len(tr), 1000)
        for e in tr[:20]:
            g.step_async(t, g.OdometryDelta(*e[:3]), m, (ks, rk)[int(e[3])], (act, ract)[int(e[3])], ctx)
        ctx.synchronize()
        ctx.mark(2)
        for e in tr[:n]:
            g.step_async(t, g.OdometryDelta(*e[:3]), m, (ks, rk)[int(e[3])], (act, ract)[int(e[3])], ctx)
        ctx.mark(3)
        ms = ctx.marks_ms(2, 3)
        g.tensor_status(t)
        out["trace_mix_hz"] = n / (ms / 1e3)
        out["trace_mix_rotation_share"] = float(tr[:n, 3].mean())
    if C <= 128:
        occ = make_floorplan(W, H, seed=0)
        js, is_ = np.nonzero(occ == 0)
        q = len(is_) // 2
        a, r = simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.3)
        f = g.DistanceField(m, ctx)
        scan = g.LidarScan(a, r, 8.0)
        cycles = []
        for _ in range(4):
            t0 = time.perf_counter()
            smp = g.dither_samples(t, 512)
            g.observation_update(t, smp, scan, m, f, g.LikelihoodParams())
            cycles.append(time.perf_counter() - t0)
        cyc = statistics.median(cycles[1:])
        step_s = 1.0 / out.get("trace_mix_hz", 1.0) if "trace_mix_hz" in out else None
        out["lidar_cycle_ms"] = cyc * 1e3
        out["lidar_samples"] = int(len(smp.cells))
        if step_s:
            out["lidar_config_hz"] = 16.0 / (16.0 * step_s + cyc)
    return out


def run_lidar(args, cfg, world, rank, local):
    """Config 3: the cmd_bench loop on the device — a step every iteration,
    and on every `lidar`-th (s % lidar == 0) the observation cycle
    dither_samples(tensor) (belief_map + Floyd-Steinberg, budget 512) and
    observation_update. value: steps/s between CUDA events on the library
    stream (host work in the cycle shows up as stream idle time); e2e: the
    same loop with synchronous gl_step calls, wall clock."""
    import paper_1910_00572_b200 as g
    W, H, C, every = cfg["W"], cfg["H"], cfg["C"], cfg["lidar"]
    ctx = g.Context(local)
    pgm = make_map_bytes(W, H)
    m = g.load_map(pgm, 250, 0.1, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    a, r = lidar_scan(W, H)
    scan = g.LidarScan(a, r, 8.0)
    lp = g.LikelihoodParams()
    samples = [0]

    def loop(n, sync):
        for s in range(n):
            (g.step if sync else g.step_async)(t, u, m, ks, act, ctx)
            if s % every == 0:
                smp = g.dither_samples(t, 512)
                g.observation_update(t, smp, scan, m, f, lp)
                samples[0] = len(smp.cells)

    loop(max(args.warmup, every + 1), False)
    ctx.synchronize()
    g.tensor_status(t)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    dist_barrier(world)
    ctx.synchronize()
    n0 = ctx.launch_count()
    ctx.time_steps(True)
    ctx.mark(0)
    loop(args.steps, False)
    ctx.mark(1)
    ms = ctx.marks_ms(0, 1)
    ctx.synchronize()
    launches = ctx.launch_count() - n0
    kern_ms, kern_n = ctx.step_times()
    ctx.time_steps(False)
    clk = clocks.stop()
    g.tensor_status(t)
    ms_max = dist_max(ms, world, "ours")
    value = world * args.steps / (ms_max / 1e3)
    # e2e over the same trajectory and length: the belief restarts from the
    # uniform state with the same warm-up (the dither's cost depends on how
    # concentrated the belief is, so another stretch would be another workload)
    n_e2e = args.steps
    del t
    t = g.init_uniform(m, C, ctx)
    loop(max(args.warmup, every + 1), False)
    ctx.synchronize()
    dist_barrier(world)
    t0 = time.perf_counter()
    loop(n_e2e, True)
    e2e_s = dist_max(time.perf_counter() - t0, world, "ours")
    e2e = world * n_e2e / e2e_s
    bytes_launch = algo_bytes(W, H, C)
    avg_kern_s = (kern_ms / max(kern_n, 1)) / 1e3
    peak, peak_src = measured_peak()
    cpu = cpu_baseline(pgm, cfg, budget_s=args.cpu_budget_s) if (rank == 0 and world == 1 and
                                                                  not args.no_cpu_baseline) else None
    if rank != 0:
        return 0
    n_obs = (args.steps + every - 1) // every
    line = {
        "metric": metric_for(W, H, C, every), "value": value, "unit": "Hz", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": "single GPU" if world == 1 else f"{world} independent replicas (one per GPU)",
        "samples_last_observation": samples[0], "noise": [0.03, 0.03, 0.012],
        "e2e": {"value": e2e, "unit": "Hz", "h2d_bytes_per_step": 16 * C + (8 * 24 * 2 + 8 * 2 * 512) // every,
                "d2h_bytes_per_step": 4 + (8 * 2 * 512 + 16) // every,
                "how": f"{n_e2e} synchronous gl_step calls with the observation cycle every {every}, wall clock, "
                       f"over the same trajectory as value (the belief restarted from uniform, same warm-up and "
                       f"step count)"},
        "roofline": {"bound": "hbm", "achieved": bytes_launch / avg_kern_s / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": bytes_launch / avg_kern_s / 1e9 / peak, "traffic": ncu_traffic("c2"),
                     "peak_source": peak_src, "bytes_per_launch": bytes_launch, "avg_kernel_ms": avg_kern_s * 1e3,
                     "launches_timed": kern_n, "kernel": "fused step (the observation cycle is latency-bound: "
                                                        "Floyd-Steinberg is a serial chain)"},
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk,
        "extras": {"observations_timed": n_obs,
                   "observation_cycle_ms": (ms_max - args.steps * avg_kern_s * 1e3) / max(n_obs, 1)},
    }
    print(json.dumps(line))
    return 0


def run_batch(args, cfg, world, rank, local):
    """Config 5: a batch of independent robots (own map, tensor) on one GPU,
    one CUDA stream per 8 robots; value = batch steps per second (every robot
    stepped once per batch step)."""
    import paper_1910_00572_b200 as g
    from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm
    W, H, C, B = cfg["W"], cfg["H"], cfg["C"], cfg["batch"]
    ctxs = [g.Context(local) for _ in range(max(1, B // 8))]
    for c in ctxs:
        c.set_channel_chunks(1)  # 8 concurrent streams fill the GPU: no chunk recompute
    robots = []
    for r in range(B):
        ctx = ctxs[r % len(ctxs)]
        m = g.load_map(write_pgm(make_floorplan(W, H, seed=100 + r + 1000 * rank)), 250, 0.1, ctx=ctx)
        ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2.0 * math.pi / C)
        robots.append((ctx, m, ks, g.make_activation(m, ks, C, ctx), g.init_uniform(m, C, ctx)))
    u = g.OdometryDelta(0.1, 0.0, 0.0)

    def batch_step():
        for ctx, m, ks, act, t in robots:
            g.step_async(t, u, m, ks, act, ctx)

    for _ in range(args.warmup):
        batch_step()
    for c in ctxs:
        c.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    dist_barrier(world)
    n0 = sum(c.launch_count() for c in ctxs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        batch_step()
    for c in ctxs:
        c.synchronize()
    dt = time.perf_counter() - t0
    clk = clocks.stop()
    for ctx, m, ks, act, t in robots:
        g.tensor_status(t)
    dt = dist_max(dt, world, "ours")
    value = world * args.steps / dt
    # e2e: every batch step enqueued through the API (motion tables in the
    # launches) and every robot's status read back to the host before the next
    n_e2e = max(1, min(args.steps, args.e2e_steps // 4))
    dist_barrier(world)
    t0 = time.perf_counter()
    by_ctx = {}
    for ctx, m, ks, act, t in robots:
        by_ctx.setdefault(id(ctx), (ctx, []))[1].append(t)
    for _ in range(n_e2e):
        batch_step()
        for ctx, ts in by_ctx.values():  # every robot's status, one round trip per context
            g.tensors_status(ts, ctx)
    e2e_s = dist_max(time.perf_counter() - t0, world, "ours")
    e2e = world * n_e2e / e2e_s
    bytes_batch = B * algo_bytes(W, H, C)
    peak, peak_src = measured_peak()
    if rank != 0:
        return 0
    print(json.dumps({
        "metric": "batch belief updates/sec (every robot stepped once) at 64 x 512^2x72", "value": value,
        "unit": "batch-Hz", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": f"{B} independent tensors per GPU on {len(ctxs)} streams",
        "timing": "host wall clock around K batch steps with device syncs",
        "e2e": {"value": e2e, "unit": "batch-Hz", "h2d_bytes_per_step": B * 16 * C, "d2h_bytes_per_step": B * 16,
                "how": f"{n_e2e} batch steps: {B} step_async calls, then every robot's status read back "
                       f"(gl_tensors_status, one round trip per context)"},
        "roofline": {"bound": "hbm", "achieved": bytes_batch * value / world / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": bytes_batch * value / world / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                     "bytes_per_launch": algo_bytes(W, H, C), "note": "aggregate over the batch's launches"},
        "cpu_baseline": None, "gpu_launches": sum(c.launch_count() for c in ctxs) - n0, "clocks": clk,
    }))
    return 0


def sharded_cpu_baseline(cfg, budget_s):
    """configs[3] cannot run on a host (the reference needs 5 tensor-sized
    FP64 buffers, ~242 GB at 4096^2x360): time the reference at
    1024^2 with the SAME channel count (same Theta = 360, H = 3 angular
    stencil) and scale its Hz by the state ratio."""
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    sub = dict(cfg, W=1024, H=1024)
    cpu = cpu_baseline(make_map_bytes(1024, 1024), sub, budget_s=budget_s, max_steps=60, one_thread_budget_s=0)
    if cpu:
        states = 1024 * 1024 * C
        cpu["note"] = (f"reference cannot hold {W}x{H}x{C} (needs {W * H * C * 40 / 1e9:.0f} GB); value = its "
                       f"1024x1024x{C} step rate scaled by states ({cpu['value']:.3f} Hz x {states}/{W * H * C})")
        cpu["scaled_from"] = f"1024x1024x{C}"
        cpu["value"] = cpu["value"] * states / (W * H * C)
    return cpu


def run_sharded(args, cfg, world, rank, local):
    """theta-slab sharding of ONE belief across the ranks (strong scaling;
    BASELINE configs[3] at 4096^2x360): per step the fused kernel on each
    slab with its halo input planes read straight from the neighbours'
    buffers over peer memory (CUDA IPC / NVLink P2P; or NCCL send/recv with
    --exchange nccl), then a MAX all-reduce of the 8-byte step max over NCCL
    on the library's stream (paper_1910_00572_b200/sharding.py). At N = 1 the
    one shard holds every channel (its halo reads wrap to its own planes)."""
    import paper_1910_00572_b200 as g
    from paper_1910_00572_b200.sharding import ThetaShard
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    ctx = g.Context(local)
    m = g.load_map(make_map_bytes(W, H), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    halo = max(1, len(ks.angular) // 2)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    single = None
    if world > 1:
        # the same workload on ONE GPU in the same run (rank 0, before its
        # shard exists, the other ranks wait): the N = 1 point of this
        # config's strong-scaling curve, measured on this box
        if rank == 0:
            t1 = g.init_uniform(m, C, ctx)
            for _ in range(3):
                g.step_async(t1, u, m, ks, act, ctx)
            ctx.synchronize()
            n1 = max(5, min(args.steps, 50))
            ctx.mark(0)
            for _ in range(n1):
                g.step_async(t1, u, m, ks, act, ctx)
            ctx.mark(1)
            single = {"value": n1 / (ctx.marks_ms(0, 1) / 1e3), "unit": "Hz", "steps": n1,
                      "how": "the unsharded step of the same belief on rank 0's GPU alone, before sharding"}
            g.tensor_status(t1)
            del t1
        dist_barrier(world)
    shard = ThetaShard(m, C, halo, rank, world, ctx, exchange=args.exchange)
    for _ in range(args.warmup):
        shard.step(u, ks, act)
    ctx.synchronize()
    shard.status()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    dist_barrier(world)
    ctx.synchronize()
    n0 = ctx.launch_count()
    ctx.time_steps(True)
    ctx.mark(0)
    for _ in range(args.steps):
        shard.step(u, ks, act)
    ctx.mark(1)
    ms = ctx.marks_ms(0, 1)
    launches = ctx.launch_count() - n0
    kern_ms, kern_n = ctx.step_times()
    ctx.time_steps(False)
    clk = clocks.stop()
    shard.status()
    ms_max = dist_max(ms, world, "ours")
    value = args.steps / (ms_max / 1e3)  # steps of the ONE sharded belief
    # e2e: the synchronous sharded step a user makes — motion table in the
    # launch, the fused kernel, the all-reduce, the finalise, and the step
    # status read back to the host on every rank — wall clock, max over ranks
    n_e2e = max(1, min(args.steps, args.e2e_steps))
    dist_barrier(world)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        shard.step(u, ks, act)
        shard.status()
    e2e_s = dist_max(time.perf_counter() - t0, world, "ours")
    n_local = shard.c_end - shard.c_begin
    bytes_launch = 2 * 8 * W * H * n_local + W * H + 8 * W * H
    avg_kern_ms = kern_ms / max(kern_n, 1)
    achieved = bytes_launch / (avg_kern_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the CPU baseline is an N = 1 figure
        cpu = sharded_cpu_baseline(cfg, args.cpu_budget_s) if W * H * C * 40 > 40e9 else \
            cpu_baseline(make_map_bytes(W, H), cfg, budget_s=args.cpu_budget_s)
    shard.close()
    if rank != 0:
        return 0
    line = {
        "metric": metric_for(W, H, C), "value": value, "unit": "Hz", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": (f"theta-slab sharding over {world} GPU(s), {n_local} channels + 2x{halo} halo planes on "
                        "rank 0; NCCL MAX all-reduce (8 B) per step; halo exchange "
                        + ("fused into the step kernel (TMA reads of the neighbours' planes over CUDA IPC / "
                           "NVLink P2P)" if args.exchange == "peer" else "by NCCL send/recv after the step")),
        "e2e": {"value": n_e2e / e2e_s, "unit": "Hz", "h2d_bytes_per_step": 16 * (n_local + 2 * halo),
                "d2h_bytes_per_step": 4,
                "how": f"{n_e2e} synchronous sharded steps (step + all-reduce + finalise, then the status read "
                       "back on every rank), wall clock, max over ranks"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic("c4") if world == 1 else None, "peak_source": peak_src,
                     "bytes_per_launch": bytes_launch, "avg_kernel_ms": avg_kern_ms, "launches_timed": kern_n,
                     "note": "rank 0's fused kernel on its slab (per-GPU roofline)"},
        "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk,
    }
    if single:
        line["extras"] = {"single_gpu_same_config": single}
    print(json.dumps(line))
    return 0


def run_ours(args, cfg, world, rank, local):
    import paper_1910_00572_b200 as g
    if args.shard or args.config == "c4":
        return run_sharded(args, cfg, world, rank, local)
    if "batch" in cfg:
        return run_batch(args, cfg, world, rank, local)
    if cfg.get("lidar"):
        return run_lidar(args, cfg, world, rank, local)
    W, H, C = cfg["W"], cfg["H"], cfg["C"]
    ctx = g.Context(local)
    pgm = make_map_bytes(W, H)
    m = g.load_map(pgm, 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)  # gridloc_main.cpp:221

    for _ in range(args.warmup):
        g.step_async(t, u, m, ks, act, ctx)
    ctx.synchronize()
    g.tensor_status(t)

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    dist_barrier(world)
    ctx.synchronize()
    n0 = ctx.launch_count()
    # per-launch kernel times over the timed region; a step shorter than the
    # ~5 us of host time an event pair costs is sampled every 8th launch
    ctx.time_steps(True, stride=1 if W * H * C >= (1 << 24) else 8)
    ctx.mark(0)
    for _ in range(args.steps):
        g.step_async(t, u, m, ks, act, ctx)
    ctx.mark(1)
    ms = ctx.marks_ms(0, 1)
    ctx.synchronize()
    launches = ctx.launch_count() - n0
    kern_ms, kern_n = ctx.step_times()
    ctx.time_steps(False)
    clk = clocks.stop()
    g.tensor_status(t)  # raises BeliefExtinguishedError like the reference
    ms_max = dist_max(ms, world, "ours")
    value = world * args.steps / (ms_max / 1e3)

    # e2e: synchronous C-ABI step per call (host motion table in, status out)
    n_e2e = max(1, min(args.steps, args.e2e_steps))
    dist_barrier(world)
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        g.step(t, u, m, ks, act, ctx)
    e2e_s = time.perf_counter() - t0
    e2e_s = dist_max(e2e_s, world, "ours")
    e2e = world * n_e2e / e2e_s

    extras = {} if args.no_extras else measure_extras(g, ctx, m, ks, act, t, cfg, args)

    bytes_launch = algo_bytes(W, H, C)
    avg_kern_s = (kern_ms / max(kern_n, 1)) / 1e3
    achieved = bytes_launch / avg_kern_s / 1e9
    peak, peak_src = measured_peak()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if W * H * C * 8 * 5 > 40e9:
            # the reference needs 5 tensor-sized FP64 buffers:
            # time it at 1024^2 with the same channel count, report states/s
            sub = dict(cfg, W=1024, H=1024)
            cpu = cpu_baseline(make_map_bytes(1024, 1024), sub, budget_s=args.cpu_budget_s)
            if cpu:
                states = 1024 * 1024 * C
                cpu["note"] = (f"reference cannot hold {W}x{H}x{C} (needs {W * H * C * 40 / 1e9:.0f} GB); "
                               f"value = its {1024}x{1024}x{C} step rate scaled by states "
                               f"({cpu['value']:.3f} Hz x {states}/{W * H * C})")
                cpu["value"] = cpu["value"] * states / (W * H * C)
        else:
            cpu = cpu_baseline(pgm, cfg, budget_s=args.cpu_budget_s)
    if rank != 0:
        return 0
    line = {
        "metric": metric_for(W, H, C), "value": value, "unit": "Hz", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_for(cfg),
        "parallelism": "single GPU" if world == 1 else f"{world} independent replicas (one per GPU)",
        "noise": [0.03, 0.03, 0.012], "kernel_path": "fused sm_100a TMA step",
        "e2e": {"value": e2e, "unit": "Hz", "h2d_bytes_per_step": 16 * C, "d2h_bytes_per_step": 4,
                "how": f"{n_e2e} synchronous gl_step calls (motion table H2D in the launch params, the step's "
                       f"status written by the finalising kernel into mapped pinned host memory), wall clock"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.config), "peak_source": peak_src,
                     "bytes_per_launch": bytes_launch, "avg_kernel_ms": avg_kern_s * 1e3, "launches_timed": kern_n},
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk,
        "extras": extras,
    }
    print(json.dumps(line))
    return 0


def spawn_ranks(args):
    """--gpus N > 1 outside torchrun: re-exec this script under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous).
    Fails loudly when fewer than N GPUs are visible."""
    import socket
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator ranks / transport visible in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execve(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="default: c2 (configs[1], 1024^2x72) at N = 1; c4 (configs[3], 4096^2x360 theta-sharded "
                         "over the N GPUs) at N > 1")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--ref-budget-s", type=float, default=90.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the trace-mix / LIDAR-cycle extras")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="sharded halo exchange: fused peer-memory reads (default) or NCCL send/recv")
    ap.add_argument("--shard", action="store_true",
                    help="theta-shard ONE belief across the ranks (strong scaling; implied by --config c4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        spawn_ranks(args)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:
        args.config = "c2" if max(world_env, args.gpus) == 1 else "c4"
    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup(args.impl)
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    try:
        if args.impl == "reference":
            if args.config == "c4":
                return run_reference_scaled(args, cfg, max(world, args.gpus), rank)
            return run_reference(args, cfg, max(world, args.gpus), rank)
        return run_ours(args, cfg, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
