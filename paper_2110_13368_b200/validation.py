"""The paper's three validation methods driven through the B200 path
(reference: /root/reference/proj/src/core/validation.{hpp,cpp}).

* Method 1 — ``run_convergence_test``: the 1-D cosine-mode problem with
  zero-flux ends (validation.cpp:17-110), solved by the CUDA sweeps.
* Method 2 — ``cross_check``: voxel-wise |a-b| <= abs + rel*max(|a|,|b|)
  (validation.cpp:112-137); the device-side version is Session.cross_check.
* Method 3 — ``write_snapshot_pgm`` / ``write_snapshot_table``: byte-identical
  P2 graymap / CSV slice writers (validation.cpp:155-228, numbers formatted
  as std::to_chars' shortest round trip, text.cpp:9-14), and
  ``run_dirichlet_mutant_check`` (validation.cpp:230-287).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

import paper_2110_13368_b200 as B

# ---- text.cpp:9-14 ----------------------------------------------------------


def format_double(v: float) -> str:
    """std::to_chars(double) shortest round trip: the fewest characters of
    printf %f or %e form that parse back to v (ties prefer %f)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    a = abs(v)
    if a == 0.0:
        return sign + "0"
    r = repr(a)  # shortest round-trip digits (same digit string as Ryu)
    mant, _, exp = r.partition("e")
    e10 = int(exp) if exp else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # value = 0.digits... -> int(digits) * 10**(e10 - len(fp)), minus stripped leading zeros
    exp_int = e10 - len(fp)
    digits = digits.rstrip("0") if digits else "0"
    exp_int += len((ip + fp).lstrip("0")) - len(digits)
    nd = len(digits)
    sci_exp = exp_int + nd - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if sci_exp < 0 else "+") + \
        f"{abs(sci_exp):02d}"
    if exp_int >= 0:
        # %f of an integral value prints its exact decimal expansion (same length).
        fixed = str(int(a))
    else:
        pos = nd + exp_int
        fixed = (digits[:pos] + "." + digits[pos:]) if pos > 0 else "0." + "0" * (-pos) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


# ---- Method 1 (validation.cpp:17-110) ---------------------------------------


def analytic_solution_1d(x: float, t: float, diffusion: float, length: float, mode: int) -> float:
    k = mode * math.pi / length
    return 1.0 + math.cos(k * x) * math.exp(-diffusion * k * k * t)


@dataclass
class ConvergenceSetup:  # validation.hpp:34-43
    length: float = 2000.0
    diffusion: float = 1000.0
    total_time: float = 10.0
    mode: int = 4
    base_dt: float = 0.5
    fine_dx: float = 2.5
    base_dx: float = 100.0
    fine_dt: float = 0.0005


@dataclass
class ConvergenceReport:  # validation.hpp:24-30
    kind: str
    steps: List[float] = field(default_factory=list)
    errors: List[float] = field(default_factory=list)
    fitted_order: float = 0.0
    band: tuple = (0.0, 0.0)
    passed: bool = False


def run_problem_1d(dt: float, dx: float, setup: ConvergenceSetup, device: int = 0) -> float:
    """validation.cpp:27-61 on the device: max |num - exact| at T/4, T/2, T."""
    nx = int(round(setup.length / dx))
    mesh = B.mesh_from_bounds(0.0, setup.length, 0.0, dx, 0.0, dx, dx, dx, dx)
    s = B.Session(mesh, 1, device)
    s.set_substrates([setup.diffusion], [0.0], dt)
    centers = [mesh.x_min + (i + 0.5) * mesh.dx for i in range(nx)]
    s.upload_field([analytic_solution_1d(x, 0.0, setup.diffusion, setup.length, setup.mode) for x in centers])
    quarter = setup.total_time / 4.0
    spq = int(round(quarter / dt))
    if spq < 1 or abs(quarter - spq * dt) > 1e-9 * quarter:
        raise ValueError("convergence setup: dt must divide T/4")
    linf = 0.0
    for q in range(1, 5):
        s.advance(spq, dt, with_sources=False)
        if q == 3:
            continue
        t = quarter * q
        f = s.download_field()
        for i in range(nx):
            exact = analytic_solution_1d(centers[i], t, setup.diffusion, setup.length, setup.mode)
            linf = max(linf, abs(f[i] - exact))
    s.close()
    return linf


def run_convergence_test(kind: str, levels: int, setup: ConvergenceSetup = None, device: int = 0):
    setup = setup or ConvergenceSetup()
    if levels < 3:
        raise ValueError("convergence study needs at least 3 refinement levels")
    rep = ConvergenceReport(kind, band=(0.8, 1.2) if kind == "temporal" else (1.7, 2.3))
    for level in range(levels):
        scale = 2.0 ** level
        dt = setup.base_dt / scale if kind == "temporal" else setup.fine_dt
        dx = setup.fine_dx if kind == "temporal" else setup.base_dx / scale
        rep.steps.append(dt if kind == "temporal" else dx)
        rep.errors.append(run_problem_1d(dt, dx, setup, device))
    if all(e > 0.0 for e in rep.errors):
        n = float(levels)
        sx = sy = sxx = sxy = 0.0
        for lvl, e in enumerate(rep.errors):
            x, y = float(lvl), math.log2(e)
            sx += x
            sy += y
            sxx += x * x
            sxy += x * y
        rep.fitted_order = -(n * sxy - sx * sy) / (n * sxx - sx * sx)
    rep.passed = all(e > 0.0 for e in rep.errors) and rep.band[0] <= rep.fitted_order <= rep.band[1]
    return rep


# ---- Method 2 (validation.cpp:112-137) --------------------------------------


@dataclass
class CrossCheckReport:
    max_abs: float = 0.0
    max_rel: float = 0.0
    worst_value_index: int = -1
    worst_voxel: int = -1
    worst_substrate: int = -1
    passed: bool = True


def cross_check(a, b, substrates: int, abs_tol: float, rel_tol: float) -> CrossCheckReport:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("cross_check fields have different shapes")
    if abs_tol < 0 or rel_tol < 0:
        raise ValueError("cross_check tolerances must be non-negative")
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        diff = np.abs(a - b)
        # std::max(|a|, |b|) returns |a| unless |a| < |b| (a NaN |a| stays)
        mag = np.where(np.abs(a) < np.abs(b), np.abs(b), np.abs(a))
        rel = np.where((diff == 0) | (mag == 0), 0.0, diff / np.where(mag == 0, 1, mag))
        fails = diff > abs_tol + rel_tol * mag
    r = CrossCheckReport()
    if diff.size:
        # Every comparison with NaN is false in the reference loop: NaN
        # differences never become the maximum and never fail the check.
        ok = ~np.isnan(diff)
        if ok.any():
            d = np.where(ok, diff, -1.0)
            i = int(np.argmax(d))
            if d[i] > 0:
                r.max_abs, r.worst_value_index = float(d[i]), i
                r.worst_voxel, r.worst_substrate = i // substrates, i % substrates
        okr = ~np.isnan(rel)
        r.max_rel = float(rel[okr].max()) if okr.any() else 0.0
        r.passed = not bool(np.any(fails))
    return r


# ---- Method 3 (validation.cpp:155-287) --------------------------------------


def _slice(field_values, mesh: B.Mesh, S: int, substrate: int, z_slice: int):
    if substrate < 0 or substrate >= S:
        raise ValueError(f"substrate index {substrate} out of range")
    if z_slice < 0 or z_slice >= mesh.nz:
        raise ValueError(f"z slice {z_slice} out of range")
    f = np.asarray(field_values, np.float64)
    if f.size != mesh.voxel_count * S:
        raise ValueError("field does not match the mesh")
    plane = mesh.nx * mesh.ny
    return f.reshape(mesh.nz, plane, S)[z_slice, :, substrate].reshape(mesh.ny, mesh.nx)


def write_snapshot_table(field_values, mesh: B.Mesh, S: int, substrate: int, z_slice: int) -> str:
    sl = _slice(field_values, mesh, S, substrate, z_slice)
    out = [f"# {mesh.nx} {mesh.ny} {mesh.nz} {S} {substrate} {z_slice}\n"]
    for j in range(mesh.ny):
        out.append(",".join(format_double(v) for v in sl[j]) + "\n")
    return "".join(out)


def write_snapshot_pgm(field_values, mesh: B.Mesh, S: int, substrate: int, z_slice: int) -> str:
    sl = _slice(field_values, mesh, S, substrate, z_slice)
    lo = hi = float(sl[0, 0])
    for v in sl.ravel():
        lo = min(lo, float(v))
        hi = max(hi, float(v))
    out = [f"P2\n{mesh.nx} {mesh.ny}\n255\n"]
    span = hi - lo
    for j in range(mesh.ny):
        row = []
        for i in range(mesh.nx):
            px = 128
            if span > 0.0:
                x = (float(sl[j, i]) - lo) / span * 255.0
                px = min(max(int(math.floor(x + 0.5)), 0), 255)  # std::lround, x >= 0
            row.append(str(px))
        out.append(" ".join(row) + "\n")
    return "".join(out)


@dataclass
class MutantCheckReport:
    clean_reproducible: bool = False
    crosscheck_detected: bool = False
    table_detected: bool = False

    @property
    def passed(self):
        return self.clean_reproducible and self.crosscheck_detected and self.table_detected


def mutant_scenario_run(mutate: bool, device: int = 0):
    """validation.cpp:244-262 on the device: 16^3, D=1000, lambda=0.1, IC 1,
    centre clamp 38 (off by one voxel when mutated), initial clamp, 100 steps."""
    mesh = B.mesh_from_bounds(-160, 160, -160, 160, -160, 160, 20, 20, 20)
    s = B.Session(mesh, 1, device)
    dt = 0.01
    s.set_substrates([1000.0], [0.1], dt)
    centre = B.nearest_voxel(mesh, [0.0, 0.0, 0.0])
    v = centre + 1 if mutate else centre  # make_off_by_one_dirichlet (validation.cpp:230-240)
    if v < mesh.voxel_count:
        s.set_dirichlet([v], [[1]], [[38.0]])
    s.upload_field(np.ones(mesh.voxel_count))
    s.apply_dirichlet_conditions()
    s.advance(100, dt, with_sources=False)
    f = s.download_field()
    s.close()
    return mesh, f


def run_dirichlet_mutant_check(device: int = 0) -> MutantCheckReport:
    mesh, a = mutant_scenario_run(False, device)
    _, b = mutant_scenario_run(False, device)
    _, m = mutant_scenario_run(True, device)
    table = lambda f: write_snapshot_table(f, mesh, 1, 0, mesh.nz // 2)  # noqa: E731
    r = MutantCheckReport()
    r.clean_reproducible = cross_check(a, b, 1, 0.0, 0.0).passed and table(a) == table(b)
    r.crosscheck_detected = not cross_check(a, m, 1, 0.0, 0.0).passed
    r.table_detected = table(a) != table(m)
    return r
