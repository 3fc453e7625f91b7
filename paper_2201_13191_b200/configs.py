"""The BASELINE.json workload configurations.

C1  60 keV cone beam, 128^3 water cylinder, 256^2 detector, 1e6 photons, split 10
C2  150 kVp, 256^3 water + 4 Al rods, 512^2 detector, 1e7 photons, split 10
C3  150 kVp, 512^3 Al body + Fe inserts ("cylinder head"), 2048^2 detector,
    1e8 photons, split 20  (the headline: BASELINE metric "1e8 photons")
C4  C3 phantom and panel, 360 angles x 1e7 photons (angle-sharded scans)
C5  correction loop: 720 angles at 2048^2, MC grid 512^2 on every 2nd angle, 1e7, split 10

Geometry per the paper's Table I: SDD 128.2 cm, SOD 86.2 cm,
pixel pitch 0.0127 * 2304 / n cm.  Seed 20240915 (REF tests/test_transport.cpp:37).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

from . import inputs as I
from . import synthetic as S

SDD, SOD = 128.2, 86.2
SEED = 20240915


def pitch(n: int) -> float:
    return 0.0127 * 2304 / n


@dataclasses.dataclass
class Workload:
    name: str
    phantom: I.VoxelPhantom
    geometry: I.ScanGeometry
    spectrum: I.Spectrum
    response: I.DetectorResponse
    config: I.SimConfig
    description: str


def _cfg(photons, split, seed=SEED):
    return I.SimConfig(photons_total=int(photons), splitting=split, roulette_survival=0.5,
                       roulette_wmin_rel=1e-3, step_voxels=1, max_interactions=50, seed=seed)


def c1(photons: Optional[int] = None, seed: int = SEED) -> Workload:
    water = I.material("water")
    ph = S.make_cylinder_phantom(128, 0.1, 5.0, 10.0, water, 1.0)
    g = I.make_circular_geometry(SDD, SOD, 256, 256, pitch(256), 1)
    return Workload("C1", ph, g, I.monochromatic_spectrum(60.0), I.detector_response(),
                    _cfg(photons or 1_000_000, 10, seed),
                    "60 keV, 128^3 water cylinder, 256x256, 1e6 photons, split 10")


def c2(photons: Optional[int] = None, seed: int = SEED) -> Workload:
    ph = S.make_rods_phantom(256, 0.05, 5.0, 10.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                             I.material("aluminum"), 2.699)
    g = I.make_circular_geometry(SDD, SOD, 512, 512, pitch(512), 1)
    return Workload("C2", ph, g, I.kramers_spectrum(150.0), I.detector_response(),
                    _cfg(photons or 10_000_000, 10, seed),
                    "150 kVp, 256^3 water+Al rods, 512x512, 1e7 photons, split 10")


def c3_phantom() -> I.VoxelPhantom:
    return S.make_cylinder_head_phantom(512, 0.025, I.material("aluminum"), 2.699,
                                        I.material("iron"), 7.874)


def c3(photons: Optional[int] = None, seed: int = SEED, n_angles: int = 1,
       phantom: Optional[I.VoxelPhantom] = None) -> Workload:
    ph = phantom if phantom is not None else c3_phantom()
    g = I.make_circular_geometry(SDD, SOD, 2048, 2048, pitch(2048), n_angles)
    return Workload("C3", ph, g, I.kramers_spectrum(150.0), I.detector_response(),
                    _cfg(photons or 100_000_000, 20, seed),
                    "150 kVp, 512^3 Al/Fe cylinder head, 2048x2048, 1e8 photons, split 20")


def c4(photons: Optional[int] = None, seed: int = SEED) -> Workload:
    w = c3(photons or 10_000_000, seed, n_angles=360)
    w.name = "C4"
    w.description = "C3 phantom/panel, 360 angles x 1e7 photons, split 20"
    return w
