"""C5 (BASELINE.json configs[4]): the iterative scatter-correction loop on one
B200 through xs_run_iterative_correction, every stage on the device.

  720 views at 2048^2 (150 kVp, the C3 512^3 Al/Fe phantom as the object),
  MC grid 512^2 on every 2nd view (360 scatter projections x 1e7 photons,
  split 10) + 720 primary projections per iteration, recon 512^3, 3 classes,
  3 iterations.

The measurement is synthesised on the device: the object's primary at 2048^2
plus its scatter, simulated by the projector itself at the MC grid (every 2nd
view, 1e7 photons, split 10), SG-smoothed, angle-interpolated and up-sampled
exactly as the loop does (so the loop's fixed point is the true object).
--offset instead adds a flat 3% of the flat field as "scatter" (round 1's
input: the loop then drifts to unphysical, speckled segmentations whose
transport cannot skip uniform blocks).  Prints the per-iteration stage times
(REF IterationReport) and, with --ref, REF's cost of the same stages on this
host's cores from bounded samples, scaled by the operation count.

usage: python tools/bench_loop.py [n_iterations] [--ref] [--offset]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import _capi as A, configs, inputs as I  # noqa: E402
from paper_2201_13191_b200.projector import ClassSpec, CorrectionConfig  # noqa: E402

n_iter = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
with_ref = "--ref" in sys.argv
offset_scatter = "--offset" in sys.argv
N_VIEWS, NU, MC, RECON = 720, 2048, 512, 512

t_setup = time.time()
w = configs.c3(n_angles=N_VIEWS)
ph, spec, resp = w.phantom, w.spectrum, w.response
g = I.make_circular_geometry(configs.SDD, configs.SOD, NU, NU, configs.pitch(NU), N_VIEWS)
al, fe = I.material("aluminum"), I.material("iron")
cfg = CorrectionConfig(n_iterations=n_iter, simulate_every_kth_angle=2, mc_nu=MC, mc_nv=MC,
                       recon_dims=(RECON, RECON, RECON), n_classes=3,
                       class_map=[ClassSpec(0, 0.0), ClassSpec(1, 2.699), ClassSpec(2, 7.874)],
                       sim=I.SimConfig(photons_total=10_000_000, splitting=10, seed=configs.SEED))

ctx = X.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
pk = A.Packed()
gp, sp = pk.geometry(g), pk.spectrum(spec)
simp = pk.config(cfg.sim)
np_full = NU * NU
raw = torch.empty((N_VIEWS, NU, NU), dtype=torch.float64, device="cuda")
# object primary for every view (device run_scan), then the flat field
ctx.upload(ph, resp)
sub = (C.c_int32 * N_VIEWS)(*range(N_VIEWS))
ctx.check(A.lib().xs_run_scan_device(ctx.h, C.byref(gp), C.byref(sp), C.byref(simp), sub, N_VIEWS, 0,
                                     C.c_void_p(raw.data_ptr()), None, None))
empty = I.make_empty_phantom(*ph.dims, ph.voxel_size, [al, fe])
ctx.upload(empty, resp)
flat = torch.empty((NU, NU), dtype=torch.float64, device="cuda")
ctx.check(A.lib().xs_primary_device(ctx.h, C.byref(gp), 0, C.byref(sp), C.byref(simp), C.c_void_p(flat.data_ptr())))
torch.cuda.synchronize()
if offset_scatter:
    raw += 0.03 * flat  # scatter-like low-frequency offset (round 1's input)
else:  # the object's own scatter, through the loop's post-processing chain
    ctx.upload(ph, resp)
    gm = I.make_circular_geometry(configs.SDD, configs.SOD, MC, MC, configs.pitch(MC), N_VIEWS)
    gmp = pk.geometry(gm)
    sub_idx = list(range(0, N_VIEWS, 2))
    ssub = (C.c_int32 * len(sub_idx))(*sub_idx)
    scat = torch.empty((len(sub_idx), MC, MC), dtype=torch.float64, device="cuda")
    ctx.check(A.lib().xs_run_scan_device(ctx.h, C.byref(gmp), C.byref(sp), C.byref(simp), ssub, len(sub_idx), 1,
                                         None, C.c_void_p(scat.data_ptr()), None))
    win, order = X.default_sg_spec(MC, MC).window, X.default_sg_spec(MC, MC).polyorder
    ctx.check(A.lib().xs_sg_smooth(ctx.h, C.c_void_p(scat.data_ptr()), C.c_void_p(scat.data_ptr()), MC, MC,
                                   len(sub_idx), win, order, 1))
    full = torch.empty((N_VIEWS, MC, MC), dtype=torch.float64, device="cuda")
    src_a = np.ascontiguousarray(np.asarray(g.angles)[sub_idx])
    tgt_a = np.ascontiguousarray(np.asarray(g.angles))
    ctx.check(A.lib().xs_interpolate_angles(ctx.h, C.c_void_p(scat.data_ptr()), A.dptr(src_a), len(sub_idx),
                                            C.c_void_p(full.data_ptr()), A.dptr(tgt_a), N_VIEWS, MC, MC, 1))
    del scat
    for v0 in range(0, N_VIEWS, 90):  # up-sample in slabs (24 GB at full size)
        up = torch.empty((90, NU, NU), dtype=torch.float64, device="cuda")
        ctx.check(A.lib().xs_upsample_image(ctx.h, C.c_void_p(full[v0:v0 + 90].data_ptr()), MC, MC, 90,
                                            C.c_void_p(up.data_ptr()), NU, NU, 1))
        raw[v0:v0 + 90] += up.clamp_(min=0.0)
        del up
    del full
    torch.cuda.synchronize()
setup_s = time.time() - t_setup

mats = [None, al, fe]
reps = (A.XsIterationReport * n_iter)()
vol = torch.empty((RECON,) * 3, dtype=torch.float32, device="cuda")
ccfg = pk.correction_config(cfg)
mptr = pk.materials(mats)
ctx.check(A.lib().xs_upload_response(ctx.h, C.byref(pk.response(resp))))
t0 = time.time()
ctx.check(A.lib().xs_run_iterative_correction(ctx.h, C.c_void_p(raw.data_ptr()), C.c_void_p(flat.data_ptr()),
                                              C.byref(gp), C.byref(sp), C.byref(ccfg), len(mats), mptr,
                                              C.c_void_p(vol.data_ptr()), None, reps, 1))
torch.cuda.synchronize()
total = time.time() - t0
R = X.projector.reports_from(reps, n_iter)
out = {"config": "C5: 720 x 2048^2 views, MC 512^2 on every 2nd view (360 x 1e7, split 10) + 720 primaries, "
                 "recon 512^3, 3 classes", "measurement": "primary + 3% flat offset" if offset_scatter else
                 "primary + the object's MC scatter through the loop's SG / interpolation / up-sampling",
       "n_iterations": n_iter, "loop_seconds": total,
       "loop_seconds_incl_initial_ln_fbp": total, "setup_seconds": setup_s,
       "peak_mem_gb": torch.cuda.max_memory_allocated() / 2 ** 30,
       "reports": [r.__dict__ for r in R]}
print(json.dumps(out))
for r in R:
    print(f"iter {r.iteration}: total {r.seconds_total:.2f} s | seg {r.seconds_segmentation:.3f} | "
          f"mc scatter {r.seconds_mc_scatter:.2f} ({r.mc_seconds_per_projection * 1e3:.1f} ms/proj) | "
          f"mc primary {r.seconds_mc_primary:.2f} | post+corr {r.seconds_postprocess:.3f} | fbp {r.seconds_fbp:.2f} | "
          f"SF {r.mean_scatter_fraction:.4f} ncc {r.ncc_to_previous:.6f} clamped {r.negative_scatter_clamped}",
          file=sys.stderr)

if with_ref:
    import oracle_lib
    ref = oracle_lib.ref()
    cores = os.cpu_count()
    est = {}
    # MC scatter: REF simulate_scatter_stats on the MC grid, bounded photon sample
    gm = I.make_circular_geometry(configs.SDD, configs.SOD, MC, MC, configs.pitch(MC), N_VIEWS)
    n = 200_000
    t = time.perf_counter()
    ref.simulate_scatter_stats(ph, gm, 0, spec, resp, I.SimConfig(photons_total=n, splitting=10, seed=1), cores)
    dt = time.perf_counter() - t
    est["mc_scatter_s"] = dt * (cfg.sim.photons_total / n) * (N_VIEWS // 2)
    t = time.perf_counter()
    ref.simulate_primary(ph, gm, 0, spec, resp, cfg.sim, cores)
    est["mc_primary_s"] = (time.perf_counter() - t) * N_VIEWS
    # FDK at 1/8 linear size (cost ~ s^3 in both terms)
    s = 8
    gs = I.make_circular_geometry(configs.SDD, configs.SOD, NU // s, NU // s, configs.pitch(NU // s), N_VIEWS)
    small = np.random.default_rng(0).random((N_VIEWS, NU // s, NU // s))
    t = time.perf_counter()
    ref.fbp_reconstruct(small, np.asarray(gs.angles), gs, (RECON // s,) * 3, X.default_voxel_size(gs, (RECON // s,) * 3))
    est["fbp_1worker_s"] = (time.perf_counter() - t) * s ** 3
    est["iteration_s"] = est["mc_scatter_s"] + est["mc_primary_s"] + est["fbp_1worker_s"]
    est["cores"] = cores
    est["note"] = ("REF stage costs on this host: scatter from 2e5 photons on 1 view with all cores "
                   "(x 1e7/2e5 x 360), primary from 1 view (x 720), FDK with REF's fbp_reconstruct "
                   "(workers=1 as in the shim) at 1/8 linear size x 512; segmentation/post-processing omitted")
    print(json.dumps({"ref_estimate": est, "speedup_per_iteration": est["iteration_s"] / R[-1].seconds_total}))
