"""Generate the file-format and input-loader fixtures from the compiled
reference (oracle/_ref/libxscat_ref.so).

Run in the build container (where /root/reference exists and `make -C oracle`
built oracle/_ref):

    python tests/golden/make_files_golden.py

Writes tests/golden/files/:
  ref_stack.xprj, ref_phantom.xvox, ref_volume.xvol   written by REF's savers
  inputs/...   material / spectrum / response / XPRJ1 / XVOX1 / XVOL1 inputs,
               valid and broken (made here from the bundled tables)
  cfg/...      run configurations (+ a small data tree they reference)
  files_golden.json   what REF's loaders return for each input: the values
               (hex doubles) or the exact error text; for each configuration
               REF's collected validation problems ({dir} = the config's
               directory).
tests/test_files.py holds the library's loaders, savers and CLI to these.
"""
import ctypes as C
import json
import pathlib
import shutil
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2201_13191_b200 import _capi as A  # noqa: E402
from paper_2201_13191_b200 import inputs as I  # noqa: E402
from paper_2201_13191_b200 import synthetic as S  # noqa: E402

OUT = HERE / "files"
REF_SO = ROOT / "oracle" / "_ref" / "libxscat_ref.so"
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, np.float64).ravel()]


def ref_lib():
    L = C.CDLL(str(REF_SO))
    L.xr_last_error.restype = C.c_char_p
    L.xr_save_stack.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, dp]
    L.xr_load_stack.argtypes = [C.c_char_p, ip, ip, ip, dp, C.c_int64]
    L.xr_save_phantom.argtypes = [C.c_char_p, C.POINTER(A.XsPhantom)]
    L.xr_load_phantom.argtypes = [C.c_char_p, C.POINTER(A.XsMaterial), C.c_int32, ip, dp, dp,
                                  C.c_void_p, C.c_void_p]
    L.xr_save_volume.argtypes = [C.c_char_p, ip, dp, C.c_void_p]
    L.xr_load_volume.argtypes = [C.c_char_p, ip, dp, C.c_void_p, C.c_int64]
    L.xr_load_material.argtypes = [C.c_char_p, dp, ip, dp, C.c_int64]
    L.xr_load_spectrum.argtypes = [C.c_char_p, dp, dp, ip, C.c_int32]
    L.xr_load_response.argtypes = [C.c_char_p, dp, dp, dp, ip, C.c_int32]
    L.xr_config_problems.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
    return L


def outcome(L, st, values=None):
    if st != 0:
        return {"ok": False, "error": L.xr_last_error().decode()}
    return {"ok": True, **(values or {})}


def main():
    assert REF_SO.exists(), "build oracle/_ref first (make -C oracle)"
    L = ref_lib()
    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "inputs").mkdir(parents=True)
    gold = {"stack": {}, "phantom": {}, "volume": {}, "material": {}, "spectrum": {}, "response": {},
            "config": {}}
    rng = np.random.default_rng(2201)

    # ---- REF-written files
    imgs = rng.random((2, 3, 5)) * 10.0 ** rng.integers(-30, 30, (2, 3, 5))
    assert L.xr_save_stack(str(OUT / "ref_stack.xprj").encode(), 5, 3, 2,
                           np.ascontiguousarray(imgs).ctypes.data_as(dp)) == 0
    gold["stack_written"] = {"nu": 5, "nv": 3, "n": 2, "images": hexs(imgs)}

    ph = S.make_rods_phantom(6, 0.4, 1.0, 2.0, I.material("water"), 1.0, 2, 0.2, 0.5,
                             I.material("iron"), 7.874)
    pk = A.Packed()
    xph = pk.phantom(ph)
    assert L.xr_save_phantom(str(OUT / "ref_phantom.xvox").encode(), C.byref(xph)) == 0, L.xr_last_error()
    gold["phantom_written"] = {"dims": list(ph.dims), "voxel_size": hexs(ph.voxel_size),
                               "origin": hexs(ph.origin), "n_materials": len(ph.materials),
                               "ids": ph.material_id.tolist(), "density": hexs(ph.density)}

    vol = (rng.random((2, 3, 4)) * 5 - 1).astype(np.float32)
    d3 = (C.c_int32 * 3)(4, 3, 2)
    vs3 = (C.c_double * 3)(0.125, 0.3, 0.7)
    assert L.xr_save_volume(str(OUT / "ref_volume.xvol").encode(), d3, vs3, vol.ctypes.data) == 0
    gold["volume_written"] = {"dims": [4, 3, 2], "voxel_size": hexs([0.125, 0.3, 0.7]),
                              "values": hexs(vol)}

    inp = OUT / "inputs"
    raw_stack = (OUT / "ref_stack.xprj").read_bytes()
    raw_ph = (OUT / "ref_phantom.xvox").read_bytes()
    raw_vol = (OUT / "ref_volume.xvol").read_bytes()

    # ---- XPRJ1 inputs
    stacks = {"ok.xprj": raw_stack, "magic.xprj": b"XPRJ2" + raw_stack[5:], "short_header.xprj": raw_stack[:11],
              "short_pixels.xprj": raw_stack[:-3], "empty.xprj": b""}
    for name, data in stacks.items():
        (inp / name).write_bytes(data)
        nu, nv, n = C.c_int32(), C.c_int32(), C.c_int32()
        buf = np.zeros(64)
        st = L.xr_load_stack(str(inp / name).encode(), C.byref(nu), C.byref(nv), C.byref(n),
                             buf.ctypes.data_as(dp), buf.size)
        gold["stack"][name] = outcome(L, st, {"nu": nu.value, "nv": nv.value, "n": n.value,
                                              "images": hexs(buf[:nu.value * nv.value * n.value])})
    gold["stack"]["missing.xprj"] = outcome(L, L.xr_load_stack(str(inp / "missing.xprj").encode(),
                                                                C.byref(C.c_int32()), C.byref(C.c_int32()),
                                                                C.byref(C.c_int32()), None, 0))

    # ---- XVOX1 inputs (loaded with k copies of water as ids 1..k)
    water = A.XsMaterial()
    pk.material(I.material("water"), water)
    nvox = 6 * 6 * 6
    bad_id = bytearray(raw_ph)
    hdr = 5 + 12 + 48 + 4
    bad_id[hdr + 7] = 9
    neg = bytearray(raw_ph)
    neg[hdr + nvox + 4 * 100: hdr + nvox + 4 * 101] = np.float32(-1.0).tobytes()
    vac = bytearray(raw_ph)
    first_vac = int(np.flatnonzero(ph.material_id == 0)[0])
    vac[hdr + nvox + 4 * first_vac: hdr + nvox + 4 * first_vac + 4] = np.float32(0.5).tobytes()
    phantoms = {"ok.xvox": (raw_ph, 2), "too_few_materials.xvox": (raw_ph, 1),
                "magic.xvox": (b"XVOX0" + raw_ph[5:], 2), "short_header.xvox": (raw_ph[:40], 2),
                "short_voxels.xvox": (raw_ph[:-1], 2), "bad_id.xvox": (bytes(bad_id), 2),
                "negative_density.xvox": (bytes(neg), 2), "vacuum_density.xvox": (bytes(vac), 2)}
    for name, (data, k) in phantoms.items():
        (inp / name).write_bytes(data)
        d = (C.c_int32 * 3)()
        v, o = (C.c_double * 3)(), (C.c_double * 3)()
        ids = np.zeros(nvox, np.uint8)
        dens = np.zeros(nvox, np.float32)
        st = L.xr_load_phantom(str(inp / name).encode(), C.byref(water), k, d, v, o, ids.ctypes.data,
                               dens.ctypes.data)
        gold["phantom"][name] = dict(outcome(L, st, {"dims": list(d), "voxel_size": hexs(list(v)),
                                                     "origin": hexs(list(o)), "ids": ids.tolist(),
                                                     "density": hexs(dens)}), files=k)

    # ---- XVOL1 inputs
    vols = {"ok.xvol": raw_vol, "magic.xvol": b"XVOLX" + raw_vol[5:], "short_data.xvol": raw_vol[:-2]}
    for name, data in vols.items():
        (inp / name).write_bytes(data)
        d = (C.c_int32 * 3)()
        v = (C.c_double * 3)()
        buf = np.zeros(24, np.float32)
        st = L.xr_load_volume(str(inp / name).encode(), d, v, buf.ctypes.data, buf.size)
        gold["volume"][name] = outcome(L, st, {"dims": list(d), "voxel_size": hexs(list(v)),
                                               "values": hexs(buf)})

    # ---- material tables: the bundled water table, then edits of it
    import tempfile
    data = I.write_reference_data(pathlib.Path(tempfile.mkdtemp()) / "data")  # (copied into cfg/ below)
    water_txt = (data / "materials" / "water.mat").read_text()
    lines = water_txt.splitlines()

    def edit(fn):
        return "\n".join(fn(list(lines))) + "\n"

    def replace_first(prefix, new):
        def f(ls):
            i = next(k for k, s in enumerate(ls) if s.startswith(prefix))
            ls[i] = new
            return ls
        return f

    def after_section(tag, new_row, k=1):
        def f(ls):
            i = ls.index(f"[{tag}]")
            ls[i + k] = new_row
            return ls
        return f

    def drop_section(tag):
        def f(ls):
            i = ls.index(f"[{tag}]")
            j = i + 1
            while j < len(ls) and not ls[j].startswith("["):
                j += 1
            return ls[:i] + ls[j:]
        return f

    mu_x0 = lines[lines.index("[mu]") + 1].split()[0]
    mats = {
        "ok.mat": water_txt,
        "comment_tabs.mat": water_txt.replace("[mu]", "  [ mu ]   # the attenuation table"),
        "unknown_section.mat": water_txt.replace("[coherent]", "[coherentx]"),
        "malformed_section.mat": water_txt.replace("[coherent]", "[coherent"),
        "unknown_key.mat": edit(lambda ls: ["colour = red"] + ls),
        "no_equals.mat": edit(lambda ls: ["just words"] + ls),
        "missing_density.mat": edit(lambda ls: [s for s in ls if not s.startswith("density")]),
        "bad_number.mat": edit(replace_first("z_eff", "z_eff = abc")),
        "partial_number.mat": edit(replace_first("z_eff", "z_eff = 10.0xyz")),
        "one_column.mat": edit(after_section("mu", mu_x0)),
        "trailing_token.mat": edit(after_section("mu", f"{mu_x0} 4078 7")),
        "nonmonotone.mat": edit(after_section("coherent", "1e9 1", k=2)),
        "negative.mat": edit(after_section("photoelectric", "1 -3")),
        "mu_zero.mat": edit(after_section("mu", f"{mu_x0} 0")),
        "s_start.mat": edit(after_section("S", "0 0.5")),
        "f_start.mat": edit(after_section("F", "0 9.5")),
        "missing_table.mat": edit(drop_section("photoelectric")),
        "bad_z.mat": edit(replace_first("z_eff", "z_eff = -1")),
    }
    for name, txt in mats.items():
        (inp / name).write_text(txt)
    for name in list(mats) + ["missing.mat"]:
        hdr2 = np.zeros(2)
        counts = np.zeros(6, np.int32)
        xy = np.zeros(20000)
        st = L.xr_load_material(str(inp / name).encode(), hdr2.ctypes.data_as(dp), counts.ctypes.data_as(ip),
                                xy.ctypes.data_as(dp), xy.size)
        gold["material"][name] = outcome(L, st, {"z_eff": hexs([hdr2[0]])[0], "density": hexs([hdr2[1]])[0],
                                                 "counts": counts.tolist(),
                                                 "xy": hexs(xy[:2 * int(counts.sum())])})

    # ---- spectra
    spec_txt = (data / "spectra" / "w200kv_2mmal.csv").read_text()
    specs = {"ok.csv": spec_txt, "nan_row.csv": "nan, 1\n" + spec_txt, "one_column.csv": spec_txt + "300\n",
             "negative.csv": "10, 1\n20, -1\n", "nonmonotone.csv": "10, 1\n10, 1\n", "zero.csv": "10, 0\n20, 0\n",
             "range.csv": "10, 1\n2000, 1\n", "empty.csv": "# nothing\n", "blanks.csv": "\n 10 , 1 \n\n20 2 # x\n"}
    for name, txt in specs.items():
        (inp / f"spec_{name}").write_text(txt)
    for name in list(specs) + ["missing.csv"]:
        e, w = np.zeros(512), np.zeros(512)
        n = C.c_int32()
        st = L.xr_load_spectrum(str(inp / f"spec_{name}").encode(), e.ctypes.data_as(dp), w.ctypes.data_as(dp),
                                C.byref(n), 512)
        gold["spectrum"][name] = outcome(L, st, {"e": hexs(e[:n.value]), "w": hexs(w[:n.value])})

    # ---- detector responses
    resp_txt = (data / "detector" / "gd2o2s_208um.csv").read_text()
    resps = {"ok.csv": resp_txt, "two_columns.csv": "10, 1\n", "dqe.csv": "10, 1.5, 5\n",
             "deposit.csv": "10, 1, 11\n", "nonmonotone.csv": "10, 1, 5\n10, 1, 5\n", "empty.csv": "\n# none\n"}
    for name, txt in resps.items():
        (inp / f"resp_{name}").write_text(txt)
    for name in list(resps) + ["missing.csv"]:
        e, q, dep = np.zeros(512), np.zeros(512), np.zeros(512)
        n = C.c_int32()
        st = L.xr_load_response(str(inp / f"resp_{name}").encode(), e.ctypes.data_as(dp), q.ctypes.data_as(dp),
                                dep.ctypes.data_as(dp), C.byref(n), 512)
        gold["response"][name] = outcome(L, st, {"e": hexs(e[:n.value]), "dqe": hexs(q[:n.value]),
                                                 "deposit": hexs(dep[:n.value])})

    # ---- run configurations (README.md:88-127 grammar), against a data tree
    cfg = OUT / "cfg"
    cfg.mkdir()
    shutil.copytree(data, cfg / "data")
    shutil.copy(OUT / "ref_phantom.xvox", cfg / "obj.xvox")
    good = """[paths]
materials_dir     = data/materials
materials         = water.mat, iron.mat   # phantom ids 1, 2 (0 = vacuum)
spectrum          = data/spectra/w200kv_2mmal.csv
detector_response = data/detector/gd2o2s_208um.csv
phantom           = obj.xvox
output_dir        = out

[geometry]
sdd_cm = 60.0
sod_cm = 40.0
det_nu = 24
det_nv = 16
pixel_pitch_cm = 0.1
n_angles = 8

[sim]
photons_total  = 20000
splitting      = 5
roulette_survival = 0.5
roulette_wmin_rel = 1e-3
step_voxels    = 1
max_interactions = 50
seed           = 1234

[correction]
n_iterations   = 3
simulate_every_kth_angle = 2
mc_nu = 12
mc_nv = 8
recon_dim = 16
n_classes = 3
class_map = air:0, water:1.0, iron:7.874

[run]
threads = 4
"""
    configs = {
        "good.ini": good,
        "missing_keys.ini": "\n".join(s for s in good.splitlines()
                                      if not s.startswith(("sdd_cm", "materials ", "phantom"))) + "\n",
        "bad_numbers.ini": good.replace("det_nu = 24", "det_nu = 24px").replace("seed           = 1234",
                                                                                 "seed = x").replace("mc_nu = 12", "mc_nu = twelve"),
        "missing_files.ini": good.replace("iron.mat", "nope.mat").replace("obj.xvox", "nothing.xvox")
                                 .replace("data/spectra", "data/nowhere"),
        "ranges.ini": good.replace("sod_cm = 40.0", "sod_cm = 70.0").replace("pixel_pitch_cm = 0.1",
                                                                              "pixel_pitch_cm = 0")
                          .replace("splitting      = 5", "splitting = 0").replace("roulette_survival = 0.5",
                                                                                   "roulette_survival = 1.5")
                          .replace("n_classes = 3", "n_classes = 5").replace("threads = 4", "threads = 0"),
        "class_map.ini": good.replace("class_map = air:0, water:1.0, iron:7.874", "class_map = air, water:1.0"),
        "no_dir.ini": good.replace("materials_dir     = data/materials", "materials_dir = data/nodir"),
        "malformed.ini": good.replace("[sim]", "[sim"),
        "no_equals.ini": good.replace("splitting      = 5", "splitting 5"),
    }
    for name, txt in configs.items():
        (cfg / name).write_text(txt)
        buf = C.create_string_buffer(1 << 16)
        st = L.xr_config_problems(str(cfg / name).encode(), buf, len(buf))
        o = outcome(L, st, {"problems": [p for p in buf.value.decode().split("\n") if p]})
        for k in ("error", "problems"):
            if k in o:
                o[k] = (o[k].replace(str(cfg), "{dir}") if isinstance(o[k], str)
                        else [p.replace(str(cfg), "{dir}") for p in o[k]])
        gold["config"][name] = o

    # paths inside messages: {out} = tests/golden/files wherever the checkout lives
    for k in ("stack", "phantom", "volume", "material", "spectrum", "response"):
        for o in gold[k].values():
            if "error" in o:
                o["error"] = o["error"].replace(str(OUT), "{out}")
    (OUT / "files_golden.json").write_text(json.dumps(gold, indent=0, sort_keys=True))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
