"""Generate the golden fixtures from the compiled reference (oracle/_ref).

Run in the build container, where /root/reference exists and
`make -C oracle` has produced oracle/_ref/libxscat_ref.so:

    python tests/golden/make_golden.py

Every array in tests/golden/ref_golden.npz is an output of the unmodified
reference library (REF = /root/reference/proj) on the inputs recorded next to
it; tests/test_oracle.py pins the C restatement (oracle/liboracle.so) to
these values bit for bit, and tests/test_gpu_*.py compare the device path
against the oracle.
"""
import hashlib
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402
from paper_2201_13191_b200 import inputs as I  # noqa: E402
from paper_2201_13191_b200 import synthetic as S  # noqa: E402

import cases  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = oracle_lib.ref()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    out = {}

    # Philox streams (rng.hpp)
    for k, (seed, a, b, p) in enumerate(cases.RNG_STREAMS):
        out[f"rng_{k}"] = ref.rng_uniform(seed, a, b, p, 40)

    # scatter: acceptance criterion 2 + polyenergetic/roulette/variance/march
    for name, make in cases.SCATTER_CASES.items():
        ph, g, angle, spec, resp, cfg = make()
        r = ref.simulate_scatter_stats(ph, g, angle, spec, resp, cfg, 4)
        out[f"scatter_{name}_image"] = r["image"]
        if r["variance"] is not None:
            out[f"scatter_{name}_variance"] = r["variance"]
        out[f"scatter_{name}_stats"] = np.array(
            [r["total"], r["total_std_error"], r["histories"]] +
            [r["ledger"][k] for k in ("initial", "escaped", "absorbed", "culled",
                                      "roulette_killed", "roulette_boost")])

    # primary
    for name, make in cases.PRIMARY_CASES.items():
        ph, g, angle, spec, resp = make()
        out[f"primary_{name}"] = ref.simulate_primary(ph, g, angle, spec, resp)

    # samplers (acceptance criterion 1 streams)
    for mat in ("water", "aluminum"):
        m = I.material(mat)
        for e in (60.0, 100.0):
            th, ph_, ap = ref.sample_compton(m, e, 0xACCE9700, 2000)
            out[f"compton_{mat}_{int(e)}"] = np.stack([th, ph_, ap])
            th, ph_ = ref.sample_rayleigh(m, e, 0xACCE9701, 2000)
            out[f"rayleigh_{mat}_{int(e)}"] = np.stack([th, ph_])
        out[f"cdf_{mat}"] = ref.f2_q2_cdf(m)

    # tracing
    ph = cases.rods(16)
    rng = np.random.default_rng(11)
    rays = []
    for _ in range(64):
        o = rng.uniform(-6, 6, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        rays.append(np.concatenate([o, d]))
    rays = np.array(rays)
    out["trace_rays"] = rays
    out["trace_tau_step1"] = np.array([ref.trace_attenuation(ph, r[:3], r[3:], 80.0, 1) for r in rays])
    out["trace_tau_step3"] = np.array([ref.trace_attenuation(ph, r[:3], r[3:], 80.0, 3) for r in rays])
    fp = []
    for k, r in enumerate(rays):
        esc, pt, vox = ref.sample_free_path(ph, r[:3], r[3:], 80.0, (k + 0.5) / len(rays))
        fp.append(np.concatenate([[float(esc)], pt, vox]))
    out["trace_free_path"] = np.array(fp)

    # post-processing
    img = np.random.default_rng(5).random((33, 40))
    out["pp_input"] = img
    out["pp_sg_7_3"] = ref.sg_smooth(img, 7, 3)
    out["pp_sg_15_2"] = ref.sg_smooth(np.random.default_rng(6).random((48, 64)), 15, 2)
    out["pp_up_80_66"] = ref.upsample_image(img, 80, 66)
    out["pp_down_20_11"] = ref.downsample_average(img, 20, 11)
    st = np.random.default_rng(7).random((6, 9, 11))
    src = np.array([0.0, 1.0, 2.0, 3.0, 4.0, 5.0])
    tgt = np.array([0.0, 0.5, 1.0, 2.25, 5.0, 5.9, 6.2])
    out["pp_interp_stack"] = st
    out["pp_interp"] = ref.interpolate_angles(st, src, tgt)
    out["pp_sg_kernels"] = np.concatenate([ref.sg_kernel(l, r, o) for (l, r, o) in cases.SG_KERNELS])

    # photon apportioning
    out["apportion_kramers150_1e8"] = ref.apportion(I.kramers_spectrum(150.0), 10**8).astype(np.uint64)
    out["apportion_mixed_1000"] = ref.apportion(cases.mixed_spectrum(), 1000).astype(np.uint64)

    # synthetic phantom generators (REF synthetic.cpp) -> checksums
    checks = {}
    for name, (kind, n, vox, params, dens) in cases.PHANTOMS.items():
        ids, den = cases.ref_phantom(ref, kind, n, vox, params, dens)
        checks[name] = (sha(ids), sha(den))
    out["phantom_names"] = np.array(list(checks))
    out["phantom_sha"] = np.array([a + ":" + b for a, b in checks.values()])

    np.savez_compressed(HERE / "ref_golden.npz", **out)
    print("wrote", HERE / "ref_golden.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
