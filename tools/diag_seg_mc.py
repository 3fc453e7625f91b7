"""Why is the MC slower on segmented recon phantoms (C5 iterations >= 2)?
Runs one loop iteration, segments its volume like iteration 2 does, and
compares walk statistics of one 512^2 scatter projection against the C3
phantom at the same geometry."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, configs, inputs as I
from paper_2201_13191_b200.projector import ClassSpec, CorrectionConfig

N_VIEWS, NU, MC, RECON = 720, 2048, 512, int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = configs.c3(n_angles=N_VIEWS)
ph, spec, resp = w.phantom, w.spectrum, w.response
g = I.make_circular_geometry(configs.SDD, configs.SOD, NU, NU, configs.pitch(NU), N_VIEWS)
gm = I.make_circular_geometry(configs.SDD, configs.SOD, MC, MC, configs.pitch(MC), N_VIEWS)
al, fe = I.material("aluminum"), I.material("iron")
cmap = [ClassSpec(0, 0.0), ClassSpec(1, 2.699), ClassSpec(2, 7.874)]
sim = I.SimConfig(photons_total=10_000_000, splitting=10, seed=configs.SEED)
cfg = CorrectionConfig(n_iterations=1, simulate_every_kth_angle=2, mc_nu=MC, mc_nv=MC,
                       recon_dims=(RECON,) * 3, n_classes=3, class_map=cmap, sim=sim)
ctx = X.Context(0)
pk = A.Packed()
gp, sp, simp = pk.geometry(g), pk.spectrum(spec), pk.config(sim)
raw = torch.empty((N_VIEWS, NU, NU), dtype=torch.float64, device="cuda")
ctx.upload(ph, resp)
sub = (C.c_int32 * N_VIEWS)(*range(N_VIEWS))
ctx.check(A.lib().xs_run_scan_device(ctx.h, C.byref(gp), C.byref(sp), C.byref(simp), sub, N_VIEWS, 0,
                                     C.c_void_p(raw.data_ptr()), None, None))
ctx.upload(I.make_empty_phantom(*ph.dims, ph.voxel_size, [al, fe]), resp)
flat = torch.empty((NU, NU), dtype=torch.float64, device="cuda")
ctx.check(A.lib().xs_primary_device(ctx.h, C.byref(gp), 0, C.byref(sp), C.byref(simp), C.c_void_p(flat.data_ptr())))
torch.cuda.synchronize()
raw += 0.03 * flat
vol = torch.empty((RECON,) * 3, dtype=torch.float32, device="cuda")
reps = (A.XsIterationReport * 1)()
ctx.check(A.lib().xs_run_iterative_correction(ctx.h, C.c_void_p(raw.data_ptr()), C.c_void_p(flat.data_ptr()),
                                              C.byref(gp), C.byref(sp), C.byref(pk.correction_config(cfg)), 3,
                                              pk.materials([None, al, fe]), C.c_void_p(vol.data_ptr()), None, reps, 1))
torch.cuda.synchronize()
v = vol.cpu().numpy()
del raw
vs = X.default_voxel_size(g, (RECON,) * 3)


def stats(name):
    pk2 = A.Packed()
    img = np.zeros(MC * MC)
    res = A.XsScatterResult()
    res.image = A.dptr(img)
    ctx.check(A.lib().xs_simulate_scatter_stats(ctx.h, C.byref(pk2.geometry(gm)), 0, C.byref(pk2.spectrum(spec)),
                                                C.byref(pk2.config(sim)), C.byref(res)))
    s = ctx.launch_stats()
    h = s["histories"]
    print(f"{name}: kernel {s['kernel_ms']:.1f} ms, walk {s['walk_ms']:.1f} ms, palette {s['palette_size']}, "
          f"fmt {s['voxel_format']}, visits/hist {(s['free_path_steps'] + s['scoring_steps']) / h:.0f}, "
          f"walk iters/hist {s['walk_iterations'] / h:.0f}, total {res.total:.4g}")


thr = X.segment_to_scene(v, vs, 3, cmap, (RECON,) * 3, [al, fe], resp, ctx=ctx)
print("thresholds", thr, "vol range", float(np.nanmin(v)), float(np.nanmax(v)))
stats("segmented iter-1 volume")
ctx.set_option("exact_walk", 1)
stats("segmented iter-1 volume, exact walk")
ctx.set_option("exact_walk", 0)
seg = X.segment_volume(v, thr, cmap, ctx=ctx)
lab = seg.labels
print("class fractions", [float((lab == k).mean()) for k in range(3)])
b = lab.reshape(RECON // 4, 4, RECON // 4, 4, RECON // 4, 4)
uni = (b.min(axis=(1, 3, 5)) == b.max(axis=(1, 3, 5)))
print("uniform 4^3 bricks", float(uni.mean()))
# a median-filtered label map's uniformity, for comparison (not used)
ctx.upload(ph, resp)
stats("C3 phantom")
ctx.set_option("exact_walk", 1)
stats("C3 phantom, exact walk")
