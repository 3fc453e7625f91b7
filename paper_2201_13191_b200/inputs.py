"""Host-side input types of the projector and the reference's input formats.

These mirror the reference's value types (REF = /root/reference/proj):
``Material``/``Table1D`` (include/xscat/material.hpp:15-32, table.hpp:15-95),
``Spectrum`` (spectrum.hpp:14-36), ``DetectorResponse``
(detector_response.hpp:11-24), ``VoxelPhantom`` (phantom.hpp:14-37),
``ScanGeometry`` (scan_geometry.hpp:20-40) and ``SimConfig``
(transport.hpp:22-31).  They hold numpy arrays and are converted to the
C-ABI structs of include/xscat_gpu.h by :mod:`._capi`.

The text-format loaders follow the reference parsers (material.cpp:129-223,
spectrum.cpp:32-60, detector_response.cpp:50-79) so a user of the reference
can keep their data files.  The bundled tables live in
``data/xscat_tables.json`` (converted from the reference's ``proj/data`` by
tools/import_reference_tables.py, exact via float.hex).
"""
from __future__ import annotations

import dataclasses
import functools
import json
import math
import pathlib
from typing import Dict, List, Optional

import numpy as np

PI = 3.14159265358979323846
DATA_DIR = pathlib.Path(__file__).resolve().parent / "data"


class XscatError(RuntimeError):
    """Base of the errors raised by this package (REF: std::runtime_error)."""


class XscatOutOfRange(XscatError, IndexError):
    """REF std::out_of_range."""


class XscatInvalidArgument(XscatError, ValueError):
    """REF std::invalid_argument."""


class XscatDomainError(XscatError, ValueError):
    """REF std::domain_error."""


# ------------------------------------------------------------------ tables
@dataclasses.dataclass
class Table1D:
    """Strictly increasing 1-D table (REF table.hpp:15-95)."""

    x: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        self.x = np.ascontiguousarray(self.x, dtype=np.float64)
        self.y = np.ascontiguousarray(self.y, dtype=np.float64)
        if self.x.shape != self.y.shape or self.x.size == 0:
            raise XscatError("table: empty or mismatched table")
        if np.any(~(self.x[1:] > self.x[:-1])):
            raise XscatError("table: non-monotone abscissa")

    def __len__(self):
        return int(self.x.size)

    def _locate(self, v: float):
        x = self.x
        if not (x[0] <= v <= x[-1]):
            raise XscatOutOfRange(f"table: query {v:f} outside [{x[0]:f}, {x[-1]:f}]")
        lo, hi = 0, x.size - 1
        while hi - lo > 1:
            mid = (lo + hi) // 2
            if x[mid] <= v:
                lo = mid
            else:
                hi = mid
        if v == x[lo]:
            return lo, True
        if v == x[hi]:
            return hi, True
        return lo, False

    def linear(self, v: float) -> float:
        i, exact = self._locate(v)
        if exact:
            return float(self.y[i])
        t = (v - self.x[i]) / (self.x[i + 1] - self.x[i])
        return float(self.y[i] + t * (self.y[i + 1] - self.y[i]))

    def loglog(self, v: float) -> float:
        """REF table.hpp:57-69 (same libm, so bit-identical to the reference)."""
        i, exact = self._locate(v)
        if exact:
            return float(self.y[i])
        x0, x1, y0, y1 = (float(self.x[i]), float(self.x[i + 1]), float(self.y[i]),
                          float(self.y[i + 1]))
        if y0 <= 0.0 or y1 <= 0.0:
            t = (v - x0) / (x1 - x0)
            return y0 + t * (y1 - y0)
        t = (math.log(v) - math.log(x0)) / (math.log(x1) - math.log(x0))
        return math.exp(math.log(y0) + t * (math.log(y1) - math.log(y0)))

    def to_json(self):
        return {"x": [float(v).hex() for v in self.x], "y": [float(v).hex() for v in self.y]}

    @staticmethod
    def from_json(d):
        return Table1D(np.array([float.fromhex(v) for v in d["x"]]),
                       np.array([float.fromhex(v) for v in d["y"]]))


# ---------------------------------------------------------------- material
_SECTIONS = ("mu", "incoherent", "coherent", "photoelectric", "S", "F")


@dataclasses.dataclass
class Material:
    """REF material.hpp:15-32 (the F^2 dq^2 CDF is derived by the library)."""

    name: str
    z_eff: float
    density_ref: float
    mu: Table1D
    sigma_incoh: Table1D
    sigma_coh: Table1D
    sigma_pe: Table1D
    s_factor: Table1D
    f_factor: Table1D

    def tables(self):
        return (self.mu, self.sigma_incoh, self.sigma_coh, self.sigma_pe, self.s_factor,
                self.f_factor)

    def to_json(self):
        return {"name": self.name, "z_eff": float(self.z_eff).hex(),
                "density": float(self.density_ref).hex(),
                **{k: t.to_json() for k, t in zip(_SECTIONS, self.tables())}}

    @staticmethod
    def from_json(d):
        t = [Table1D.from_json(d[k]) for k in _SECTIONS]
        return Material(d["name"], float.fromhex(d["z_eff"]), float.fromhex(d["density"]), *t)


def _invariant(name, what):
    raise XscatError(f"material '{name}': invariant violation: {what}")


def validate_material(m: Material) -> None:
    """REF validate_material (material.cpp:57-103)."""
    if not m.name:
        _invariant("(unnamed)", "missing name")
    if not m.z_eff > 0.0:
        _invariant(m.name, "z_eff must be > 0")
    if not m.density_ref > 0.0:
        _invariant(m.name, "density must be > 0")
    for tag, t in zip(_SECTIONS, m.tables()):
        if np.any(~(t.y >= 0.0)) or not np.all(np.isfinite(t.y)):
            _invariant(m.name, f"negative or non-finite value in [{tag}]")
    if np.any(~(m.mu.y > 0.0)):
        _invariant(m.name, "mu values must be > 0")
    sq, sv = m.s_factor.x, m.s_factor.y
    if sq[0] != 0.0 or sv[0] != 0.0:
        _invariant(m.name, "S table must start at S(0) = 0")
    if np.any(sv[1:] < sv[:-1]):
        _invariant(m.name, "S must be non-decreasing in q")
    if sv[-1] > m.z_eff * (1.0 + 1e-9):
        _invariant(m.name, "S must not exceed z_eff")
    fq, fv = m.f_factor.x, m.f_factor.y
    if fq[0] != 0.0:
        _invariant(m.name, "F table must start at q = 0")
    if abs(fv[0] - m.z_eff) > 1e-9 * m.z_eff:
        _invariant(m.name, "F(0) must equal z_eff")
    if np.any(fv[1:] > fv[:-1] * (1.0 + 1e-12) + 1e-15):
        _invariant(m.name, "F must be non-increasing in q")


def load_material(path) -> Material:
    """Parse REF's plain-text material format (material.cpp:129-223)."""
    path = pathlib.Path(path)
    try:
        lines = path.read_text().splitlines()
    except OSError:
        raise XscatError(f"cannot open material file {path}")
    header: Dict[str, str] = {}
    tables: Dict[str, List[List[float]]] = {}
    section = None
    for no, raw in enumerate(lines, 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            if not line.endswith("]"):
                raise XscatError(f"{path}:{no}: parse error: malformed section header")
            section = line[1:-1].strip()
            if section not in _SECTIONS:
                raise XscatError(f"{path}:{no}: parse error: unknown section [{section}]")
            continue
        if section is None:
            if "=" not in line:
                raise XscatError(f"{path}:{no}: parse error: expected key=value before first section")
            k, v = (s.strip() for s in line.split("=", 1))
            if k not in ("name", "z_eff", "density"):
                raise XscatError(f"{path}:{no}: parse error: unknown header key '{k}'")
            header[k] = v
            continue
        parts = line.split()
        if len(parts) != 2:
            raise XscatError(f"{path}:{no}: parse error: expected two numeric columns")
        tables.setdefault(section, [[], []])
        tables[section][0].append(float(parts[0]))
        tables[section][1].append(float(parts[1]))
    if not all(k in header for k in ("name", "z_eff", "density")):
        raise XscatError(f"{path}:{len(lines)}: parse error: missing header key (name=, z_eff=, density=)")
    name = header["name"]
    for tag in _SECTIONS:
        if tag not in tables:
            _invariant(name, f"missing table [{tag}]")
        xs = tables[tag][0]
        if any(not (b > a) for a, b in zip(xs, xs[1:])):
            _invariant(name, f"non-monotone abscissa in [{tag}]")
    m = Material(name, float(header["z_eff"]), float(header["density"]),
                 *[Table1D(np.array(tables[t][0]), np.array(tables[t][1])) for t in _SECTIONS])
    validate_material(m)
    return m


def mu_at(m: Material, energy_kev: float, density: float) -> float:
    """REF mu_at (material.cpp:246-251)."""
    if not density >= 0.0:
        raise XscatInvalidArgument("mu_at: negative density")
    return m.mu.loglog(energy_kev) * density


# ---------------------------------------------------------------- spectrum
@dataclasses.dataclass
class Spectrum:
    """REF spectrum.hpp:14-36."""

    energy_kev: np.ndarray
    weight: np.ndarray

    def __post_init__(self):
        self.energy_kev = np.ascontiguousarray(self.energy_kev, dtype=np.float64)
        self.weight = np.ascontiguousarray(self.weight, dtype=np.float64)

    @property
    def n_bins(self):
        return int(self.energy_kev.size)

    def total_weight(self):
        s = 0.0
        for w in self.weight:
            s += float(w)
        return s

    def to_json(self):
        return {"e": [float(v).hex() for v in self.energy_kev],
                "w": [float(v).hex() for v in self.weight]}

    @staticmethod
    def from_json(d):
        return Spectrum(np.array([float.fromhex(v) for v in d["e"]]),
                        np.array([float.fromhex(v) for v in d["w"]]))


def monochromatic_spectrum(energy_kev: float, weight: float = 1.0) -> Spectrum:
    return Spectrum(np.array([energy_kev]), np.array([weight]))


def validate_spectrum(s: Spectrum) -> None:
    """REF validate_spectrum (spectrum.cpp:11-30)."""
    if s.n_bins == 0:
        raise XscatError("spectrum: no bins")
    if not (np.all(np.isfinite(s.energy_kev)) and np.all(np.isfinite(s.weight))):
        raise XscatError("spectrum: non-finite entry")
    if np.any(~(s.weight >= 0.0)):
        raise XscatError("spectrum: negative weight")
    if np.any(~(s.energy_kev[1:] > s.energy_kev[:-1])):
        raise XscatError("spectrum: non-monotone abscissa")
    if not s.total_weight() > 0.0:
        raise XscatError("spectrum: all weights zero")
    if s.energy_kev[0] < 1.0 or s.energy_kev[-1] > 1000.0:
        raise XscatError("spectrum: energies must lie within [1 keV, 1 MeV]")


def _csv_rows(path, ncol, what):
    rows = []
    for no, raw in enumerate(pathlib.Path(path).read_text().splitlines(), 1):
        line = raw.split("#", 1)[0].replace(",", " ").split()
        if not line:
            continue
        if len(line) < ncol:
            raise XscatError(f"{path}:{no}: expected {what}")
        rows.append([float(v) for v in line[:ncol]])
    return rows


def load_spectrum(path) -> Spectrum:
    """REF load_spectrum (spectrum.cpp:32-60): two-column CSV (keV, weight)."""
    rows = _csv_rows(path, 2, "two columns (keV, weight)")
    s = Spectrum(np.array([r[0] for r in rows]), np.array([r[1] for r in rows]))
    validate_spectrum(s)
    return s


# ------------------------------------------------------- detector response
@dataclasses.dataclass
class DetectorResponse:
    """REF detector_response.hpp:11-24."""

    dqe: Table1D
    deposit: Table1D

    def response_factor(self, energy_kev: float) -> float:
        return self.deposit.linear(energy_kev) / energy_kev

    def to_json(self):
        return {"dqe": self.dqe.to_json(), "deposit": self.deposit.to_json()}

    @staticmethod
    def from_json(d):
        return DetectorResponse(Table1D.from_json(d["dqe"]), Table1D.from_json(d["deposit"]))


def load_detector_response(path) -> DetectorResponse:
    """REF load_detector_response (detector_response.cpp:50-79)."""
    rows = _csv_rows(path, 3, "three columns (keV, dqe, deposit_keV)")
    if not rows:
        raise XscatError(f"{path}: empty detector response")
    e = np.array([r[0] for r in rows])
    r = DetectorResponse(Table1D(e, np.array([r[1] for r in rows])),
                         Table1D(e, np.array([r[2] for r in rows])))
    if np.any(~((r.dqe.y >= 0) & (r.dqe.y <= 1))):
        raise XscatError("detector response: dqe outside [0,1]")
    if np.any(r.deposit.y > r.deposit.x * (1.0 + 1e-12)):
        raise XscatError("detector response: deposit exceeds incident energy")
    return r


# ------------------------------------------------------------------ phantom
@dataclasses.dataclass
class VoxelPhantom:
    """REF VoxelPhantom (phantom.hpp:14-37): x-fastest u8 ids + f32 densities.

    ``materials[0]`` is the vacuum sentinel (``None``)."""

    dims: tuple
    voxel_size: tuple
    origin: tuple
    material_id: np.ndarray
    density: np.ndarray
    materials: List[Optional[Material]]

    def __post_init__(self):
        self.dims = tuple(int(v) for v in self.dims)
        self.voxel_size = tuple(float(v) for v in self.voxel_size)
        self.origin = tuple(float(v) for v in self.origin)
        self.material_id = np.ascontiguousarray(self.material_id, dtype=np.uint8).reshape(-1)
        self.density = np.ascontiguousarray(self.density, dtype=np.float32).reshape(-1)

    def voxel_count(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    def index(self, ix, iy, iz):
        return ix + self.dims[0] * (iy + self.dims[1] * iz)


def make_empty_phantom(nx, ny, nz, voxel_size, materials) -> VoxelPhantom:
    """REF make_empty_phantom (phantom.cpp:16-31); vacuum prepended at id 0."""
    vs = tuple(float(v) for v in voxel_size)
    origin = ((-nx * vs[0]) * 0.5, (-ny * vs[1]) * 0.5, (-nz * vs[2]) * 0.5)
    n = nx * ny * nz
    mats = list(materials)
    if not mats or mats[0] is not None:
        mats = [None] + mats
    return VoxelPhantom((nx, ny, nz), vs, origin, np.zeros(n, np.uint8), np.zeros(n, np.float32),
                        mats)


def validate_phantom(ph: VoxelPhantom) -> None:
    """REF validate_phantom (phantom.cpp:33-56)."""
    if min(ph.dims) <= 0:
        raise XscatError("phantom: dims must be positive")
    if not min(ph.voxel_size) > 0.0:
        raise XscatError("phantom: voxel size must be positive")
    n = ph.voxel_count()
    if ph.material_id.size != n or ph.density.size != n:
        raise XscatError("phantom: array size mismatch")
    if not ph.materials:
        raise XscatError("phantom: no material table")
    top = int(ph.material_id.max()) if n else 0
    if top >= len(ph.materials):
        raise XscatError(f"phantom: material id {top} has no loaded material")
    if np.any(~(ph.density >= 0.0)):
        raise XscatError("phantom: negative density")
    if np.any((ph.material_id == 0) & (ph.density != 0.0)):
        raise XscatError("phantom: vacuum voxel with nonzero density")


# ----------------------------------------------------------------- geometry
@dataclasses.dataclass
class ScanGeometry:
    """REF ScanGeometry (scan_geometry.hpp:20-40)."""

    sdd: float
    sod: float
    nu: int
    nv: int
    pixel_pitch: float
    angles: np.ndarray

    def __post_init__(self):
        self.angles = np.ascontiguousarray(self.angles, dtype=np.float64)

    @property
    def n_angles(self):
        return int(self.angles.size)

    def detector_area(self):
        return self.nu * self.nv * self.pixel_pitch * self.pixel_pitch

    def source_position(self, i):
        a = float(self.angles[i])
        return np.array([self.sod * math.cos(a), self.sod * math.sin(a), 0.0])

    def detector_center(self, i):
        a = float(self.angles[i])
        r = self.sdd - self.sod
        return np.array([-r * math.cos(a), -r * math.sin(a), 0.0])

    def detector_u_axis(self, i):
        a = float(self.angles[i])
        return np.array([-math.sin(a), math.cos(a), 0.0])

    def pixel_position(self, i, u, v):
        """REF scan_geometry.cpp:69-77 (same expression order)."""
        c, ua = self.detector_center(i), self.detector_u_axis(i)
        du = (u + 0.5 - 0.5 * self.nu) * self.pixel_pitch
        dv = (v + 0.5 - 0.5 * self.nv) * self.pixel_pitch
        return c + ua * du + np.array([0.0, 0.0, 1.0]) * dv

    def with_grid(self, nu, nv, pixel_pitch):
        return ScanGeometry(self.sdd, self.sod, nu, nv, pixel_pitch, self.angles.copy())


def validate_geometry(g: ScanGeometry) -> None:
    """REF validate_geometry (scan_geometry.cpp:9-26)."""
    if not (g.sod > 0.0 and g.sdd > g.sod):
        raise XscatError("geometry: require 0 < sod < sdd")
    if g.nu <= 0 or g.nv <= 0:
        raise XscatError("geometry: detector pixel counts must be positive")
    if not g.pixel_pitch > 0.0:
        raise XscatError("geometry: pixel pitch must be positive")
    if g.n_angles == 0:
        raise XscatError("geometry: no angles")
    a = g.angles
    if np.any(a < 0.0) or np.any(a >= 2.0 * PI):
        raise XscatError("geometry: angles must lie in [0, 2pi)")
    if np.any(~(a[1:] > a[:-1])):
        raise XscatError("geometry: angles must be strictly increasing")


def make_circular_geometry(sdd, sod, nu, nv, pixel_pitch, n_angles) -> ScanGeometry:
    """REF make_circular_geometry (scan_geometry.cpp:28-42)."""
    angles = np.array([2.0 * PI * i / n_angles for i in range(n_angles)])
    g = ScanGeometry(float(sdd), float(sod), int(nu), int(nv), float(pixel_pitch), angles)
    validate_geometry(g)
    return g


# ------------------------------------------------------------------- config
@dataclasses.dataclass
class SimConfig:
    """REF SimConfig (transport.hpp:22-31), same defaults."""

    photons_total: int = 10000
    splitting: int = 1
    roulette_survival: float = 0.5
    roulette_wmin_rel: float = 1e-3
    step_voxels: int = 1
    max_interactions: int = 50
    seed: int = 0
    track_variance: bool = False


def validate_sim_config(c: SimConfig) -> None:
    """REF validate_sim_config (transport.cpp:26-40)."""
    if c.photons_total < 1:
        raise XscatError("sim config: photons_total must be >= 1")
    if c.splitting < 1:
        raise XscatError("sim config: splitting must be >= 1")
    if not (0.0 < c.roulette_survival <= 1.0):
        raise XscatError("sim config: roulette_survival must lie in (0,1]")
    if c.roulette_wmin_rel < 0.0:
        raise XscatError("sim config: roulette_wmin_rel must be >= 0")
    if c.step_voxels < 1:
        raise XscatError("sim config: step_voxels must be >= 1")
    if c.max_interactions < 1:
        raise XscatError("sim config: max_interactions must be >= 1")


# ------------------------------------------------------------ bundled data
@functools.lru_cache(maxsize=None)
def _bundle():
    return json.loads((DATA_DIR / "xscat_tables.json").read_text())


def material(name: str) -> Material:
    """Bundled material by name: water, aluminum, iron, cement, gd2o2s."""
    return Material.from_json(_bundle()["materials"][name])


def spectrum(name: str) -> Spectrum:
    """Bundled spectrum: w200kv_2mmal, mono_60kev, mono_100kev."""
    return Spectrum.from_json(_bundle()["spectra"][name])


def detector_response(name: str = "gd2o2s_208um") -> DetectorResponse:
    return DetectorResponse.from_json(_bundle()["detector"][name])


def kramers_spectrum(e_max: float, filter_material: Optional[Material] = None,
                     filter_cm: float = 0.2, e_min: float = 20.0, step: float = 2.0) -> Spectrum:
    """Kramers bremsstrahlung behind an aluminium filter, peak-normalised.

    The reference's own recipe (tools/make_material_tables.cpp:341-357, used for
    its 200 kV spectrum); BASELINE configs 2-4 use it with e_max = 150 (65 bins)."""
    al = filter_material or material("aluminum")
    e_list, w_list = [], []
    e = e_min
    while e <= e_max - 2.0:
        kramers = (e_max - e) / e
        filt = math.exp(-mu_at(al, e, al.density_ref) * filter_cm)
        e_list.append(e)
        w_list.append(kramers * filt)
        e += step
    peak = 0.0
    for w in w_list:
        peak = max(peak, w)
    return Spectrum(np.array(e_list), np.array([w / peak for w in w_list]))


# ------------------------------------------------ writers of REF's formats
def save_material(m: Material, path) -> None:
    """REF save_material (material.cpp:225-244): %.17g round-trips exactly."""
    lines = [f"name = {m.name}", f"z_eff = {float(m.z_eff):.17g}",
             f"density = {float(m.density_ref):.17g}"]
    for tag, t in zip(_SECTIONS, m.tables()):
        lines.append(f"[{tag}]")
        lines += [f"{float(x):.17g} {float(y):.17g}" for x, y in zip(t.x, t.y)]
    pathlib.Path(path).write_text("\n".join(lines) + "\n")


def save_spectrum(s: Spectrum, path) -> None:
    """REF save_spectrum (spectrum.cpp:62-73)."""
    rows = ["# keV, relative fluence"] + [f"{float(e):.17g}, {float(w):.17g}"
                                         for e, w in zip(s.energy_kev, s.weight)]
    pathlib.Path(path).write_text("\n".join(rows) + "\n")


def save_detector_response(r: DetectorResponse, path) -> None:
    """REF save_detector_response (detector_response.cpp:81-89)."""
    rows = ["# keV, dqe, deposit_keV"] + [f"{float(e):.17g}, {float(q):.17g}, {float(d):.17g}"
                                         for e, q, d in zip(r.dqe.x, r.dqe.y, r.deposit.y)]
    pathlib.Path(path).write_text("\n".join(rows) + "\n")


def write_reference_data(root) -> pathlib.Path:
    """Recreate the reference's proj/data tree (materials/, spectra/,
    detector/) from the bundled tables, for programs that load REF files."""
    root = pathlib.Path(root)
    b = _bundle()
    for sub in ("materials", "spectra", "detector"):
        (root / sub).mkdir(parents=True, exist_ok=True)
    for name in b["materials"]:
        save_material(material(name), root / "materials" / f"{name}.mat")
    for name in b["spectra"]:
        save_spectrum(spectrum(name), root / "spectra" / f"{name}.csv")
    for name in b["detector"]:
        save_detector_response(detector_response(name), root / "detector" / f"{name}.csv")
    return root
