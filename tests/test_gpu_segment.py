"""Segmentation stage on the device against the C
oracle (pinned bit-exact to REF in tests/test_segment.py), and the device
phantom upload against the host one: same thresholds, labels, phantoms,
device grids and scatter images, bit for bit."""
import ctypes as C

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200.projector import ClassSpec

from cases import poly, rods
from test_segment import mixture

pytestmark = pytest.mark.gpu


def bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


@pytest.mark.parametrize("n_classes", [2, 3, 4])
@pytest.mark.parametrize("bins,shape", [(64, (20, 21, 22)), (1024, (37, 41, 29)), (4096, (64, 64, 64))])
def test_otsu_bitwise(orc, n_classes, bins, shape):
    vol = mixture(np.random.default_rng(7 * n_classes + bins), shape, nan=True)
    assert np.array_equal(bits(X.otsu_thresholds(vol, n_classes, bins)), bits(orc.otsu_thresholds(vol, n_classes, bins)))


def test_otsu_errors():
    vol = np.full((16, 16, 16), 4.0, np.float32)
    with pytest.raises(I.XscatError, match="degenerate histogram"):
        X.otsu_thresholds(vol, 2)
    with pytest.raises(I.XscatInvalidArgument, match="n_classes must be in"):
        X.otsu_thresholds(vol, 5)
    with pytest.raises(I.XscatInvalidArgument, match="too few histogram bins"):
        X.otsu_thresholds(vol, 3, 2)


def test_segment_volume_bitwise(orc):
    vol = mixture(np.random.default_rng(3), (33, 20, 17), nan=True)
    thr = [17.5, 35.25]
    cmap = [ClassSpec(), ClassSpec(1, 1.0), ClassSpec(2, 2.0)]
    seg = X.segment_volume(vol, thr, cmap)
    assert np.array_equal(seg.labels, orc.segment_volume(vol, thr, 3))
    with pytest.raises(I.XscatError, match="strictly increasing"):
        X.segment_volume(vol, [3.0, 3.0], cmap)
    with pytest.raises(I.XscatError, match="class_map must cover all 3 classes"):
        X.segment_volume(vol, thr, cmap[:2])


@pytest.mark.parametrize("src,tgt", [((8, 8, 8), (4, 4, 4)), ((13, 11, 9), (5, 4, 3)),
                                     ((40, 36, 30), (40, 36, 30)), ((64, 64, 48), (32, 16, 48))])
def test_density_phantom_bitwise(orc, src, tgt):
    rng = np.random.default_rng(sum(src) + sum(tgt))
    labels = rng.integers(0, 3, size=src[::-1]).astype(np.uint8)
    cmap = [ClassSpec(0, 0.0), ClassSpec(1, 0.9), ClassSpec(2, 2.699)]
    mats = [I.material("water"), I.material("aluminum")]
    seg = X.SegmentationResult([], labels, cmap)
    ph = X.to_density_phantom(labels, (0.1, 0.1, 0.1), seg, tgt, mats)
    ids, dens = orc.to_density_phantom(labels, cmap, tgt, mats)
    assert np.array_equal(ph.material_id, ids)
    assert np.array_equal(ph.density.view(np.uint32), dens.view(np.uint32))
    bad = labels.copy()
    bad.reshape(-1)[5] = 9
    with pytest.raises(I.XscatError, match="unmapped label 9"):
        X.to_density_phantom(bad, (0.1, 0.1, 0.1), X.SegmentationResult([], bad, cmap), tgt, mats)


def _device_phantom(ph):
    """(xs_phantom with device arrays, keep-alive tensors)."""
    import torch
    ids = torch.from_numpy(np.ascontiguousarray(ph.material_id)).cuda()
    dens = torch.from_numpy(np.ascontiguousarray(ph.density)).cuda()
    torch.cuda.synchronize()
    pk = A.Packed()
    p = pk.phantom(ph)
    p.material_id = C.cast(C.c_void_p(ids.data_ptr()), C.POINTER(C.c_uint8))
    p.density = C.cast(C.c_void_p(dens.data_ptr()), C.POINTER(C.c_float))
    return p, (pk, ids, dens)


def _scatter(ctx, g, angle, spec, cfg):
    pk = A.Packed()
    img = np.zeros(g.nu * g.nv)
    res = A.XsScatterResult()
    res.image = A.dptr(img)
    ctx.check(A.lib().xs_simulate_scatter_stats(ctx.h, C.byref(pk.geometry(g)), angle, C.byref(pk.spectrum(spec)),
                                                C.byref(pk.config(cfg)), C.byref(res)))
    return img, res.total


@pytest.mark.parametrize("kind", ["palette", "raw"])
def test_device_upload_matches_host_upload(kind):
    ph, g, angle, spec, resp, cfg = poly()
    if kind == "raw":  # > 255 distinct (material, density) pairs: the raw format
        ph.density = ph.density * (1.0 + 1e-3 * (np.arange(ph.density.size) % 300)).astype(np.float32)
        ph.density[ph.material_id == 0] = 0.0
    ctx = X.Context(0)
    ctx.set_option("upload_path", 0)  # the host encoder
    ctx.upload(ph, resp)
    a = _scatter(ctx, g, angle, spec, cfg)
    host_fmt = ctx.launch_stats()["voxel_format"]
    p, keep = _device_phantom(ph)
    ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))
    b = _scatter(ctx, g, angle, spec, cfg)
    # raw for > 255 pairs; else the 8-bit palette, or 4-bit codes when the voxel walk is chosen
    assert ctx.launch_stats()["voxel_format"] == host_fmt and (host_fmt == 2) == (kind == "raw")
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    ctx.close()


def test_device_upload_validation_errors():
    ph = rods(16)
    ctx = X.Context(0)
    ph.density[100] = 0.5
    ph.material_id[100] = 0
    p, keep = _device_phantom(ph)
    with pytest.raises(I.XscatError, match="vacuum voxel with nonzero density"):
        ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))
    ph = rods(16)
    ph.material_id[7] = 9
    p, keep = _device_phantom(ph)
    with pytest.raises(I.XscatError, match="material id 9 has no loaded material"):
        ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))
    ctx.close()


def test_segment_to_scene_matches_host_chain(orc):
    """FDK-like volume -> fused device stage vs oracle chain + host upload."""
    ph0, g, angle, spec, resp, cfg = poly()
    nz, ny, nx = 24, 32, 32
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    r2 = (x - 15.5) ** 2 + (y - 15.5) ** 2
    rng = np.random.default_rng(11)
    vol = np.where(r2 < 14 ** 2, 19.0, 0.2) + np.where((x - 20) ** 2 + (y - 12) ** 2 < 9, 40.0, 0.0)
    vol = (vol + rng.normal(0.0, 0.7, vol.shape)).astype(np.float32)
    voxel = (0.3, 0.3, 0.3)
    cmap = [ClassSpec(0, 0.0), ClassSpec(1, 1.0), ClassSpec(3, 7.874)]
    mats = [I.material("water"), I.material("aluminum"), I.material("iron")]
    ctx = X.Context(0)
    thr = X.segment_to_scene(vol, voxel, 3, cmap, (nx, ny, nz), mats, resp, ctx=ctx)
    assert np.array_equal(bits(thr), bits(orc.otsu_thresholds(vol, 3, 1024)))
    dev = _scatter(ctx, g, angle, spec, cfg)
    labels = orc.segment_volume(vol, thr, 3)
    ids, dens = orc.to_density_phantom(labels, cmap, (nx, ny, nz), mats)
    vs = tuple(voxel[a] * vol.shape[2 - a] / (nx, ny, nz)[a] for a in range(3))
    ph = I.VoxelPhantom((nx, ny, nz), vs, tuple(-n * v * 0.5 for n, v in zip((nx, ny, nz), vs)), ids, dens,
                        [None] + mats)
    ctx2 = X.Context(0)
    ctx2.set_option("upload_path", 0)
    ctx2.upload(ph, resp)
    host = _scatter(ctx2, g, angle, spec, cfg)
    assert dev[1] > 0 and np.array_equal(dev[0], host[0]) and dev[1] == host[1]
    ctx.close()
    ctx2.close()


def test_walk_mode_is_chosen_per_phantom():
    """walk_mode 2 (default): the upload probe keeps the block walk on a
    blocky phantom and the voxel walk on a speckled one; each choice gives the
    same image as forcing that mode."""
    ph, g, angle, spec, resp, cfg = poly()
    rng = np.random.default_rng(9)
    speckled = I.VoxelPhantom(ph.dims, ph.voxel_size, ph.origin, ph.material_id.copy(), ph.density.copy(),
                              ph.materials)
    flip = (rng.uniform(size=ph.material_id.size) < 0.3) & (ph.material_id > 0)
    speckled.material_id[flip] = 2
    speckled.density[flip] = 7.874
    for phantom, want in ((ph, 1), (speckled, 0)):
        ctx = X.Context(0)
        ctx.upload(phantom, resp)
        auto = _scatter(ctx, g, angle, spec, cfg)
        assert ctx.launch_stats()["block_walk"] == want
        ctx.set_option("walk_mode", want)
        forced = _scatter(ctx, g, angle, spec, cfg)
        assert np.array_equal(auto[0], forced[0])
        ctx.close()


@pytest.mark.parametrize("kind", ["palette", "raw"])
def test_staged_upload_matches_host_encoder(kind):
    """xs_upload_phantom's default path (pinned staging + device encode) gives
    the host encoder's grid: identical scatter images; same validation errors."""
    ph, g, angle, spec, resp, cfg = poly()
    if kind == "raw":
        ph.density = ph.density * (1.0 + 1e-3 * (np.arange(ph.density.size) % 300)).astype(np.float32)
        ph.density[ph.material_id == 0] = 0.0
    out = []
    for path in (0, 1):
        ctx = X.Context(0)
        ctx.set_option("upload_path", path)
        ctx.upload(ph, resp)
        out.append(_scatter(ctx, g, angle, spec, cfg))
        bad = rods(16)
        bad.density[100], bad.material_id[100] = 0.5, 0
        with pytest.raises(I.XscatError, match="vacuum voxel with nonzero density"):
            ctx.upload(bad, resp)
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


def _pinned(ph):
    """The phantom with its id / density arrays in page-locked host memory."""
    import dataclasses
    import torch
    ids = torch.from_numpy(np.ascontiguousarray(ph.material_id)).pin_memory().numpy()
    dens = torch.from_numpy(np.ascontiguousarray(ph.density)).pin_memory().numpy()
    return dataclasses.replace(ph, material_id=ids, density=dens)


def test_pinned_and_multi_chunk_uploads_match_host_encoder():
    """xs_upload_phantom with caller-pinned arrays (straight DMA) and with a
    phantom of several 8M-voxel staging chunks (the pinned ring, 2.6 chunks)
    gives the host encoder's grid: identical primary and scatter images."""
    ph, g, angle, spec, resp, cfg = poly()
    zi = np.arange(336) * 32 // 336  # 32^3 -> 256 x 256 x 336 (x fastest), same extent
    up = lambda a: a.reshape(32, 32, 32).repeat(8, 1).repeat(8, 2)[zi].reshape(-1)
    vs = ph.voxel_size
    big = I.VoxelPhantom((256, 256, 336), (vs[0] / 8, vs[1] / 8, vs[2] * 32 / 336), ph.origin,
                         up(ph.material_id), up(ph.density), ph.materials)
    for phantom in (ph, big):
        out = []
        for path, arrays in ((0, phantom), (1, phantom), (1, _pinned(phantom))):
            ctx = X.Context(0)
            ctx.set_option("upload_path", path)
            prim = X.Projector(arrays, resp, ctx=ctx).primary(g, angle, spec)  # (uploads)
            out.append((prim, *_scatter(ctx, g, angle, spec, cfg)))
            ctx.close()
        for o in out[1:]:
            assert np.array_equal(o[0], out[0][0]) and np.array_equal(o[1], out[0][1]) and o[2] == out[0][2]
    bad = _pinned(rods(16))
    bad.density[100], bad.material_id[100] = 0.5, 0
    ctx = X.Context(0)
    with pytest.raises(I.XscatError, match="vacuum voxel with nonzero density"):
        ctx.upload(bad, resp)
    ctx.close()
