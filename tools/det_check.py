import sys, pathlib, shutil, subprocess, tempfile, os
sys.path.insert(0, '.')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import files as F, inputs as I
CFG = pathlib.Path('tests/golden/files/cfg')
work = pathlib.Path(tempfile.mkdtemp()) / 'cfg'; shutil.copytree(CFG, work)
mats = [F.load_material(work / 'data/materials' / f) for f in ('water.mat', 'iron.mat')]
ph = F.load_phantom(work / 'obj.xvox', mats)
spec = F.load_spectrum(work / 'data/spectra/w200kv_2mmal.csv')
resp = F.load_detector_response(work / 'data/detector/gd2o2s_208um.csv')
g = I.make_circular_geometry(60.0, 40.0, 24, 16, 0.1, 8)
cfg = I.SimConfig(photons_total=20000, splitting=5, seed=99)
ref = None; bad = 0
for i in range(15):
    p = X.Projector(ph, resp, ctx=X.Context(0))
    s = p.run_scan(g, spec, cfg, [0, 5], X.SCATTER).scatter.images
    if ref is None: ref = s
    elif not np.array_equal(ref, s): bad += 1; print('in-process mismatch', i, np.abs(ref - s).max())
for i in range(8):
    r = subprocess.run(['paper_2201_13191_b200/bin/xscat_b200', 'simulate', '--config', str(work / 'good.ini'), '--what', 'scatter', '--angles', '0,5', '--seed', '99'], capture_output=True, text=True)
    if r.returncode: print('cli rc', r.returncode, r.stderr); continue
    got = F.load_stack(work / 'out/scatter.xprj').images
    if not np.array_equal(got, ref.astype(np.float32).astype(np.float64)): bad += 1; print('cli mismatch', i, np.abs(got - ref).max(), r.stdout)
print('done bad', bad)
