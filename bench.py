"""Benchmark of the B200 Monte Carlo scatter projector (driver contract).

One step = one projection of BASELINE config C3: 150 kVp, 512^3 Al/Fe
"cylinder head" phantom, 2048x2048 flat panel, 1e8 photon histories,
splitting 20 (BASELINE.json metric "photon histories/sec and sec/projection
(1e8 photons)").  Every step goes through the library's multi-GPU entry
point xs_simulate_scatter_stats_mgpu: with N GPUs (torchrun, one process per
GPU) the projection's history range is split into N contiguous photon batches
(one per rank) whose fixed-point tallies are summed by an ncclReduce inside
libxscatgpu (its own communicator, xs_ctx_comm_init) onto rank 0, which
finalizes the image (strong scaling: total work fixed).  Results are
bit-identical for every N.

  value : histories/s with the scene resident on the device (kernel path)
  e2e   : the same through the C ABI with page-locked host buffers: phantom
          upload (H2D + device validation and encode) and image D2H inside
          every step
  --impl reference : the reference CPU implementation (oracle/_ref, compiled
          from the reference sources) on this host's cores, bounded sample.
"""
import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "photon histories/sec and sec/projection (1e8 photons) at 1/2/4/8 B200 vs CPU"
UNIT = "histories/s"
WORKLOAD = ("C3: 150 kVp (65 bins), 512^3 Al body + Fe inserts (cylinder head), 2048x2048 "
            "flat panel, 1e8 photon histories per projection, splitting 20")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [v for v in sm if mx and v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_for(name, photons=None, phantom=None):
    """SURVEY.md 8(d) workloads: C1 / C2 (the smaller parity configs), C3 (the
    BASELINE metric's projection, the default)."""
    from paper_2201_13191_b200 import configs
    if name == "c1":
        return configs.c1(photons=photons)
    if name == "c2":
        return configs.c2(photons=photons)
    return configs.c3(photons=photons, phantom=phantom)


def workload_text(w):
    if w.name == "C3":
        return WORKLOAD
    return f"{w.name}: {w.description}"


def cpu_reference_rate(budget_s=15.0, calib=4000, reps=2, workload="c3"):
    """REF simulate_scatter_stats on this host's cores (bounded sample of the
    workload's projection, C3 by default):
    the sample grows until one call takes >= budget/2, then `reps` more calls
    of that size give the rate (histories / their summed time), the way the
    reference arm times its steps."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib  # test infrastructure: the CPU baseline leg only
    from paper_2201_13191_b200 import configs
    from paper_2201_13191_b200 import _capi as A
    import ctypes as C
    import numpy as np

    ref = oracle_lib.ref()
    kind = "reference"
    lib = ref
    if ref is None:
        lib = oracle_lib.oracle()
        kind = "port"
    cores = os.cpu_count() or 1
    import dataclasses
    w = workload_for(workload, calib)
    w_full = workload_for(workload, None, phantom=w.phantom)
    W = w.name

    def cfg_of(n):
        return dataclasses.replace(w.config, photons_total=int(n))

    pk = A.Packed()
    ph, resp = pk.phantom(w.phantom), pk.response(w.response)
    g, spec = pk.geometry(w.geometry), pk.spectrum(w.spectrum)
    img = np.zeros(w.geometry.nu * w.geometry.nv)

    if kind == "reference":
        scene = lib.L.xr_scene_create(C.byref(ph), C.byref(resp))

        def run(n):
            cfg = pk.config(cfg_of(n))
            res = A.XsScatterResult()
            res.image = A.dptr(img)
            t = time.perf_counter()
            st = lib.L.xr_scene_simulate_scatter(scene, C.byref(g), 0, C.byref(spec), C.byref(cfg),
                                                 cores, C.byref(res))
            dt = time.perf_counter() - t
            assert st == 0, lib.fn("last_error")()
            return dt, res.histories
    else:
        def run(n):
            cfg = cfg_of(n)
            t = time.perf_counter()
            r = lib.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, cfg,
                                           cores)
            return time.perf_counter() - t, r["histories"]

    # grow the sample until one call takes >= budget/2 (REF's fixed per-call
    # cost, 64 chunk images of 2048^2 fp64, is then amortised like at 1e8)
    n = calib
    dt, h = run(n)
    while dt < 0.5 * budget_s and n < 20_000_000:
        n = int(n * min(16.0, max(2.0, budget_s / max(dt, 1e-3))))
        dt, h = run(n)
    samples = [run(n) for _ in range(reps)] if reps > 0 else [(dt, h)]
    T, H = sum(d for d, _ in samples), sum(x for _, x in samples)
    rates = [x / d for d, x in samples]
    return {"value": H / T, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{W} scene (bounded sample): {len(samples)} calls of {samples[0][1]} of "
                      f"{w_full.config.photons_total:.0e} histories, {T:.1f} s with {cores} threads (per call "
                      f"{min(rates):.3g}-{max(rates):.3g} hist/s); includes REF's fixed 64-chunk "
                      f"{w.geometry.nu}^2 image cost"}, \
        (kind, lib, run, n)


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    base, (kind, lib, run, n) = cpu_reference_rate(budget_s=args.ref_seconds, reps=0,
                                                    workload=args.workload)
    w = workload_for(args.workload, 1000)
    for _ in range(args.warmup):
        run(max(1000, n // 4))
    times, hist = [], 0
    for _ in range(args.steps):
        dt, h = run(n)
        times.append(dt)
        hist += h
    value = hist / sum(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_text(w), "histories_per_step": n, "sampled": True},
            "sec_per_projection": workload_for(args.workload, None, phantom=w.phantom).config.photons_total / value,
            "cpu_baseline": {**base, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_13191_b200 as X
    from paper_2201_13191_b200 import _capi as A
    from paper_2201_13191_b200 import configs

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    torch.cuda.set_device(device)

    t0 = time.time()
    w = workload_for(args.workload, args.photons)
    g, spec, cfg, resp = w.geometry, w.spectrum, w.config, w.response
    cfg.step_voxels = args.step
    log(f"[rank {rank}] scene built in {time.time() - t0:.1f}s")
    ctx = X.Context(device)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    proj = X.Projector(w.phantom, resp, ctx=ctx)
    # the library's own NCCL communicator (xs_ctx_comm_init): rank 0 makes the
    # id, torch.distributed only carries its 128 bytes to the other ranks
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(X.Context.comm_unique_id()), dtype=torch.uint8))
    if ws > 1:
        dist.broadcast(uid, src=0)
    ctx.comm_init(ws, rank, bytes(uid.cpu().numpy().tobytes()))
    n_hist = X.history_count(spec, cfg.photons_total)
    image = torch.empty(g.nu * g.nv, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        # xs_simulate_scatter_stats_mgpu: this rank's photon batch, ncclReduce of the
        # fixed-point accumulators onto rank 0, finalize into a device image there
        r = proj.scatter_stats_mgpu(g, 0, spec, cfg, root=0, d_image_ptr=image.data_ptr(),
                                    host_image=False)
        ls = r.stats
        kms = (ls["kernel_ms"], ls["walk_ms"], ls["launches"] + 1)  # + the finalize kernel
        stats = None
        if rank == 0:
            stats = dict(ls)
            stats["total"] = r.total
            stats["total_std_error"] = r.total_std_error
        return kms, stats

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(device)
    sampler.start()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    ev = []
    kernel_ms, steps_total = [], 0
    last = None
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed iterations (outside the events)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        kms, st = step()
        b.record(stream)
        ev.append((a, b))
        kernel_ms.append(kms)
        if st:
            last = st
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_rank = torch.tensor([sum(step_ms), sum(k[0] for k in kernel_ms) / len(kernel_ms),
                           sum(k[1] for k in kernel_ms) / len(kernel_ms)], dtype=torch.float64,
                          device="cuda")
    if ws > 1:
        dist.all_reduce(t_rank, op=dist.ReduceOp.MAX)
    total_ms, kernel_ms_max, walk_ms_max = float(t_rank[0]), float(t_rank[1]), float(t_rank[2])
    launches = sum(k[2] for k in kernel_ms)
    ms_per_step = total_ms / args.steps
    value = n_hist / (ms_per_step / 1e3)

    # ---------------- primary image of the same projection (reported beside the scatter
    # metric: "Primary is timed and reported separately")
    primary_ms = None
    if rank == 0:
        proj.primary(g, 0, spec, cfg)  # warm
        torch.cuda.synchronize()
        pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pa.record(stream)
        for _ in range(3):
            proj.primary(g, 0, spec, cfg)
        pb.record(stream)
        torch.cuda.synchronize()
        primary_ms = pa.elapsed_time(pb) / 3

    # ---------------- e2e: C ABI with host buffers (phantom upload + image D2H each step)
    e2e = None
    if not args.no_e2e:
        # the caller's host buffers are page-locked (allocated once, outside
        # the timed region): the phantom's id / density arrays and the image
        import dataclasses
        ph_h = dataclasses.replace(
            w.phantom, material_id=torch.from_numpy(w.phantom.material_id).pin_memory().numpy(),
            density=torch.from_numpy(w.phantom.density).pin_memory().numpy())
        img_h = torch.empty(g.nu * g.nv, dtype=torch.float64).pin_memory().numpy()
        n_e2e = max(1, min(args.steps, 3))

        def e2e_step():
            pk = A.Packed()
            A.check(A.lib().xs_upload_phantom(ctx.h, A.C.byref(pk.phantom(ph_h))), ctx.h)
            # the image lands in the caller's host buffer (img_h, reused)
            proj.scatter_stats_mgpu(g, 0, spec, cfg, root=0, host_image=rank == 0,
                                    image_out=img_h if rank == 0 else None)
            torch.cuda.synchronize()

        e2e_step()
        if ws > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        if ws > 1:
            dist.barrier()
        dt = torch.tensor([(time.perf_counter() - t) / n_e2e], dtype=torch.float64, device="cuda")
        if ws > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        vox_bytes = int(ctx.launch_stats()["upload_bytes"])  # encoded grid copied H2D
        e2e = {"value": n_hist / float(dt[0]), "unit": UNIT,
               "h2d_bytes_per_step": vox_bytes,
               "d2h_bytes_per_step": int(img_h.nbytes) if rank == 0 else 0,
               "steps": n_e2e,
               "note": "per step: xs_upload_phantom of the host u8 id + f32 density grid "
                       "(page-locked host arrays: H2D, device validation + palette encode), then "
                       "xs_simulate_scatter_stats_mgpu with a host image: this rank's photon "
                       "batch, ncclReduce, finalize, image D2H on rank 0"}

    # ---------------- per-kernel device times of one projection, untimed: one
    # pipeline (the two pipelines' kernels overlap, so their summed event
    # intervals are not kernel durations) with CUDA events around every
    # kernel of every wave (XSCAT_KTIME, on the launching streams)
    kernels = None
    if rank == 0 and not args.no_ktime:
        os.environ["XSCAT_KTIME"] = "1"
        ctx.set_option("wave_pipes", 1)
        proj.scatter_stats(g, 0, spec, cfg)
        ks = proj.scatter_stats(g, 0, spec, cfg).stats
        ctx.set_option("wave_pipes", 2)
        del os.environ["XSCAT_KTIME"]
        names = ("setup_ms", "walk_ms", "score_ms", "event_ms", "admit_ms")
        tot = sum(ks[k] for k in names)
        kernels = {"pipelines": 1, "transport_ms": ks["kernel_ms"],
                   **{k: ks[k] for k in names},
                   "shares": {k[:-3]: ks[k] / tot for k in names},
                   "walk_iterations_per_history": ks["walk_iterations"] / ks["histories"],
                   "walk_lane_occupancy": ks["walk_iterations"] / max(1, ks["walk_lane_slots"]),
                   "uniform_block_share": ks["uniform_iterations"] / max(1, ks["walk_iterations"])}

    if rank == 0:
        hbm, kind = peaks()
        steps_vox = (last or {}).get("free_path_steps", 0) + (last or {}).get("scoring_steps", 0)
        alg_bytes = 5.0 * steps_vox  # REF voxel layout: u8 id + f32 density per visit
        # dominant kernel = the walk (every voxel visit happens there): its
        # device time over the projection's waves, CUDA events on the launching
        # stream -- from the one-pipeline pass (a kernel duration); else the
        # timed two-pipeline sum (inflated by the overlap)
        walk_s = (kernels["walk_ms"] if kernels else walk_ms_max) / 1e3
        achieved = alg_bytes / walk_s / 1e9 if walk_s > 0 else 0.0
        traffic, prof = None, {}
        tp = ROOT / "profiles" / "bench_kernel_ncu.json"
        if tp.exists() and w.name == "C3":  # the committed ncu capture is of the C3 walk
            try:
                prof = json.loads(tp.read_text())
                traffic = prof.get("walk_dram_bytes_per_projection")
            except Exception:
                prof = {}
        # the walk is issue-bound: warp instructions per iteration and issue
        # utilisation from the committed ncu capture of the same kernel, the
        # iteration count from this run (device counters)
        issue = None
        if kernels and prof.get("walk_warp_instructions_per_warp_iteration"):
            it = kernels["walk_iterations_per_history"] * n_hist
            warp_it = it / max(kernels["walk_lane_occupancy"], 1e-9) / 32.0
            wi = warp_it * prof["walk_warp_instructions_per_warp_iteration"]
            clk = (clocks.get("sm_mhz") or prof.get("sm_mhz") or 1965.0) * 1e6
            peak_issue = 148 * 4 * clk  # warp instructions per second (4 schedulers / SM)
            issue = {"achieved_warp_inst_per_s": wi / walk_s, "peak_warp_inst_per_s": peak_issue,
                     "frac": wi / walk_s / peak_issue,
                     "warp_instructions_per_warp_iteration": prof["walk_warp_instructions_per_warp_iteration"],
                     "ncu_issue_active": prof.get("walk_issue_active_pct"),
                     "note": "walk warp instructions = device-counted iterations / lane occupancy / 32 "
                             "x instructions per warp iteration (ncu, profiles/bench_kernel_ncu.json)"}
        cpu = None
        if ws == 1 and not args.no_cpu:
            try:
                cpu, _ = cpu_reference_rate(budget_s=args.cpu_seconds, workload=args.workload)
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_text(w) + (f", step_voxels {args.step} (march)" if args.step > 1 else ""),
                       "histories": n_hist, "splitting": cfg.splitting,
                       "detector": [g.nu, g.nv], "phantom": list(w.phantom.dims),
                       "parallelism": (f"photon batches x{ws}, ncclReduce of the fixed-point tallies "
                                       "inside libxscatgpu (xs_simulate_scatter_stats_mgpu)") if ws > 1
                       else "1 GPU (xs_simulate_scatter_stats_mgpu, 1 rank)",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "sec_per_projection": ms_per_step / 1e3,
            "primary_ms": primary_ms,
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_kind": kind,
                         "kernel": "wave_walk (every wave of one projection, one pipeline)",
                         "algorithmic_bytes_per_projection": alg_bytes,
                         "voxel_visits_per_projection": steps_vox,
                         "walk_ms": walk_s * 1e3, "walk_ms_two_pipelines_summed": walk_ms_max,
                         "transport_ms": kernel_ms_max,
                         "kernels": kernels,
                         "issue": issue,
                         "walker_state_dram_share": prof.get("walker_state_dram_share"),
                         "note": "5 B per REF voxel visit (u8 id + f32 density, SURVEY.md 8(d)) / "
                                 "walk-kernel time; traffic = ncu DRAM bytes of the same walk "
                                 "launches, mostly walker-state streaming. The device grid is an "
                                 "8-bit palette (1 B/voxel) with uniform blocks and same-code runs "
                                 "crossed without loads, so the REF byte model does not bind (frac "
                                 "> 1 means the walk crosses REF's voxel visits faster than HBM "
                                 "could stream REF's bytes for them): the walk is issue-bound, see "
                                 "'issue' (achieved / peak warp instructions per second)"},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "wall_s": wall,
            "result": {"total": (last or {}).get("total"),
                       "total_std_error": (last or {}).get("total_std_error")},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def c4_arm(args):
    """C4 (BASELINE configs[3]): a full scan, 360 angles x 1e7 photons on the C3
    phantom and panel, sharded by angle across the ranks (contiguous angle
    ranges, no collective; total work is fixed: strong scaling).  One step =
    the whole scan."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_13191_b200 as X
    from paper_2201_13191_b200 import configs

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    n_ang = args.angles
    w = configs.c4(photons=args.photons if args.photons != int(1e8) else 10_000_000)
    g = X.inputs.make_circular_geometry(configs.SDD, configs.SOD, 2048, 2048, configs.pitch(2048), n_ang)
    mine = list(range(n_ang * rank // ws, n_ang * (rank + 1) // ws))
    ctx = X.Context(local)
    proj = X.Projector(w.phantom, w.response, ctx=ctx)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(X.Context.comm_unique_id()), dtype=torch.uint8))
    if ws > 1:
        dist.broadcast(uid, src=0)
    ctx.comm_init(ws, rank, bytes(uid.cpu().numpy().tobytes()))
    # the caller's host output (this rank's images), allocated and touched once
    scat = np.empty((n_ang, 2048, 2048))
    scat[mine[0]:mine[-1] + 1] = 0.0
    for _ in range(args.warmup):
        proj.run_scan(g, w.spectrum, w.config, mine[:1], X.SCATTER)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    t = time.perf_counter()
    for _ in range(args.steps):
        # xs_run_scan_mgpu: this rank's contiguous angle range, images to its host memory
        proj.run_scan_mgpu(g, w.spectrum, w.config, list(range(n_ang)), X.SCATTER, gather=False,
                           scatter_out=scat)
    torch.cuda.synchronize()
    dt = torch.tensor([(time.perf_counter() - t) / args.steps], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    clocks = sampler.stop()
    n_hist = X.history_count(w.spectrum, w.config.photons_total) * n_ang
    if rank == 0:
        sec = float(dt[0])
        print(json.dumps({
            "metric": METRIC, "value": n_hist / sec, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4: full scan, {n_ang} angles x {w.config.photons_total:.0e} photons, C3 "
                                   "phantom and 2048^2 panel, splitting 20, angle-sharded",
                       "parallelism": f"angles x{ws}", "l2": "inputs (134 MB grid + 3.5 GB walker state) exceed L2"},
            "sec_per_projection": sec / n_ang * ws,
            "e2e": {"value": n_hist / sec, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 8 * 2048 * 2048 * len(mine),
                    "note": "xs_run_scan_mgpu through the C ABI (angle-sharded, no gather), scatter "
                            "images copied to each rank's host memory every angle"},
            "clocks": clocks}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--photons", type=float, default=None,
                    help="histories per step (default: the workload's, 1e8 for C3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ktime", action="store_true", help="skip the untimed per-kernel timing pass")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4"],
                    help="c3: one 1e8-photon projection (the BASELINE metric); c1 / c2: the smaller "
                         "SURVEY.md 8(d) projections; c4: angle-sharded full scan")
    ap.add_argument("--angles", type=int, default=360)
    ap.add_argument("--step", type=int, default=1,
                    help="SimConfig.step_voxels (REF's march mode for > 1, trace.cpp:116-134; "
                         "the paper's production setting is 2-3, PAPER.md:920-933)")
    args = ap.parse_args()
    args.photons = int(args.photons) if args.photons else None
    if args.impl == "reference":
        return reference_arm(args)
    if args.workload == "c4":
        return c4_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
