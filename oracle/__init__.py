"""TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA product path.

Two independent CPU implementations of the hot path, used by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm only:

* ``Oracle``: ctypes over ``_build/liboracle.so``, the plain-C restatement in
  ``biodiff_oracle.c`` (each function cites the reference file:line it follows).
* ``Reference``: ctypes over ``_ref/libbiodiff_ref.so``, the UNMODIFIED
  reference sources (/root/reference/proj/src/core) compiled by the Makefile
  here plus the ``ref_shim.cpp`` driver. Absent when the reference could not
  be built (the prebuilt .so travels to the GPU box with the snapshot).

Nothing in paper_2110_13368_b200/ imports this package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbiodiff_ref.so")
REF_SOURCES = "/root/reference/proj/src/core"

_P = ctypes.POINTER
_d = ctypes.c_double
_i64 = ctypes.c_int64
_u8 = ctypes.c_uint8
_vp = ctypes.c_void_p


def build(quiet: bool = True):
    """Builds liboracle.so always, and the reference .so when its sources exist."""
    targets = ["oracle"] + (["ref", "binding"] if os.path.isdir(REF_SOURCES) else [])
    subprocess.run(["make", "-C", HERE, "-j8"] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _dp(a):
    return a.ctypes.data_as(_P(_d))


def _ip(a):
    return a.ctypes.data_as(_P(_i64))


def _f(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_precompute.argtypes = [ctypes.c_int, ctypes.c_int, _P(_d), _P(_d), _d, _d, ctypes.c_int,
                                     _P(_d), _P(_d), _P(_d)]
        L.orc_sweep.argtypes = [_P(_d), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _P(_d), _P(_d), _P(_d)]
        L.orc_dirichlet.argtypes = [_P(_d), ctypes.c_int, _i64, _P(_i64), _P(_u8), _P(_d)]
        L.orc_nearest_voxel.argtypes = [_P(_d), _P(_d), _P(ctypes.c_int), _P(_d)]
        L.orc_nearest_voxel.restype = _i64
        L.orc_group.argtypes = [_i64, _P(_i64), _P(_d), _P(_d), _P(_d), _P(ctypes.c_int), _P(_i64), _P(_i64),
                                _P(_i64)]
        L.orc_group.restype = _i64
        L.orc_sources.argtypes = [_P(_d), ctypes.c_int, _i64, _P(_i64), _P(_i64), _P(_i64), _P(_d), _P(_d),
                                  _P(_d), _P(_d), _d, _d]
        _oracle = L
    return _oracle


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if os.path.isdir(REF_SOURCES):
                build()
            else:
                raise FileNotFoundError(f"{REF_SO} not built and the reference sources are absent")
        L = ctypes.CDLL(REF_SO)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_create.argtypes = [_P(_d), _P(_d), ctypes.c_int, _P(_d), _P(_d), _P(_d), ctypes.c_int, ctypes.c_int,
                                 _P(_vp)]
        L.ref_destroy.argtypes = [_vp]
        L.ref_mesh_dims.argtypes = [_vp, _P(ctypes.c_int)]
        L.ref_set_field.argtypes = [_vp, _P(_d), _i64]
        L.ref_get_field.argtypes = [_vp, _P(_d), _i64]
        L.ref_get_field_range.argtypes = [_vp, _i64, _i64, _P(_d)]
        L.ref_add_dirichlet.argtypes = [_vp, _i64, _P(_i64), _P(_u8), _P(_d)]
        L.ref_dirichlet_size.argtypes = [_vp]
        L.ref_dirichlet_size.restype = _i64
        L.ref_get_dirichlet.argtypes = [_vp, _P(_i64), _P(_u8), _P(_d)]
        L.ref_add_boundary_dirichlet.argtypes = [_vp, _P(_u8), _P(_d)]
        L.ref_set_agents.argtypes = [_vp, _i64, _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d), _P(_d)]
        L.ref_group_count.argtypes = [_vp]
        L.ref_group_count.restype = _i64
        L.ref_get_grouping.argtypes = [_vp, _P(_i64), _P(_i64), _P(_i64)]
        L.ref_build_workspaces.argtypes = [_vp, _d]
        L.ref_get_workspace.argtypes = [_vp, ctypes.c_int, _P(_d), _P(_d), _P(_d), _P(ctypes.c_int)]
        L.ref_sweep.argtypes = [_vp, ctypes.c_int]
        L.ref_apply_dirichlet.argtypes = [_vp]
        L.ref_diffuse_decay_step.argtypes = [_vp]
        L.ref_sources_step.argtypes = [_vp, _d]
        L.ref_run.argtypes = [_vp, _i64, _d, ctypes.c_int, _P(_d)]
        L.ref_convergence.argtypes = [ctypes.c_int, ctypes.c_int, _P(_d), _P(_d), _P(_d), _P(ctypes.c_int)]
        L.ref_mutant_check.argtypes = [_P(ctypes.c_int)]
        L.ref_format_double.argtypes = [_d, ctypes.c_char_p, ctypes.c_int]
        L.ref_format_int.argtypes = [_i64, ctypes.c_char_p, ctypes.c_int]
        L.ref_cross_check.argtypes = [_P(_d), _P(_d), _i64, ctypes.c_int, _d, _d, _P(_d), _P(_d), _P(_i64),
                                      _P(ctypes.c_int)]
        L.ref_translate_vector_to_array.argtypes = [_P(_P(_d)), _P(_i64), _i64, _P(_d), _P(ctypes.c_int)]
        L.ref_translate_round_trip.argtypes = [_P(_d), _i64, ctypes.c_int, _P(_d)]
        L.ref_load_agents.argtypes = [_vp, ctypes.c_char_p, _P(ctypes.c_char_p), ctypes.c_int]
        L.ref_agent_count.argtypes = [_vp]
        L.ref_agent_count.restype = _i64
        L.ref_get_agents.argtypes = [_vp, _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d), _P(_d)]
        L.ref_snapshot.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _i64]
        L.ref_snapshot.restype = _i64
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _rchk(code):
    if code != 0:
        raise RefError(code, ref_lib().ref_last_error().decode())


def field_sha256(read_range, count: int, chunk: int = 1 << 25) -> str:
    """SHA-256 of a float64 field's little-endian bytes, read in pieces:
    read_range(offset, n, out) fills out[:n] with values[offset, offset+n).
    Fixes the full-length / full-size parity runs in tests/golden/digests.json
    without holding two copies of a 34 GB field."""
    import hashlib
    h = hashlib.sha256()
    buf = np.empty(min(chunk, max(count, 1)), np.float64)
    for off in range(0, count, chunk):
        n = min(chunk, count - off)
        read_range(off, n, buf)
        h.update(buf[:n].astype("<f8", copy=False).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------------------
# The C restatement (biodiff_oracle.c)
# --------------------------------------------------------------------------
class Oracle:
    """Single-threaded C restatement driven from numpy arrays."""

    @staticmethod
    def precompute(n, D, lam, h, dt, dims):
        D = _f(D)
        lam = _f(lam)
        S = D.size
        q = np.zeros(S)
        dinv = np.zeros(n * S)
        cb = np.zeros(n * S)
        rc = oracle_lib().orc_precompute(n, S, _dp(D), _dp(lam), h, dt, dims, _dp(q), _dp(dinv), _dp(cb))
        if rc:
            raise ValueError("invalid precompute arguments")
        return q, dinv, cb

    @staticmethod
    def workspaces(shape, h, D, lam, dt):
        nx, ny, nz = shape
        dims = 1 + (ny > 1) + (nz > 1)
        ws = {0: Oracle.precompute(nx, D, lam, h[0], dt, dims)}
        if ny > 1:
            ws[1] = Oracle.precompute(ny, D, lam, h[1], dt, dims)
        if nz > 1:
            ws[2] = Oracle.precompute(nz, D, lam, h[2], dt, dims)
        return ws

    @staticmethod
    def sweep(rho, shape, S, axis, ws):
        q, dinv, cb = ws
        oracle_lib().orc_sweep(_dp(rho), shape[0], shape[1], shape[2], S, axis, _dp(q), _dp(dinv), _dp(cb))

    @staticmethod
    def dirichlet(rho, S, voxels, mask, values):
        v = _i(voxels)
        m = np.ascontiguousarray(np.asarray(mask, np.uint8))
        x = _f(values)
        oracle_lib().orc_dirichlet(_dp(rho), S, v.size, _ip(v), m.ctypes.data_as(_P(_u8)), _dp(x))

    @staticmethod
    def group(ids, positions, bounds, h, shape):
        ids = _i(ids)
        pos = _f(positions)
        n = ids.size
        gv = np.zeros(max(n, 1), np.int64)
        go = np.zeros(n + 1, np.int64)
        order = np.zeros(max(n, 1), np.int64)
        b = _f(bounds)
        hh = _f(h)
        sh = np.ascontiguousarray(np.asarray(shape, np.int32))
        G = oracle_lib().orc_group(n, _ip(ids), _dp(pos), _dp(b), _dp(hh), sh.ctypes.data_as(_P(ctypes.c_int)),
                                   _ip(gv), _ip(go), _ip(order))
        if G < 0:
            raise ValueError("agent outside the domain")
        return gv[:G].copy(), go[:G + 1].copy(), order[:n].copy()

    @staticmethod
    def sources(rho, S, grouping, volume, sec, upt, sat, dt, inv_voxel_volume):
        gv, go, order = grouping
        vol = _f(volume)
        se, up, sa = _f(sec), _f(upt), _f(sat)
        oracle_lib().orc_sources(_dp(rho), S, gv.size, _ip(gv), _ip(go), _ip(order), _dp(vol), _dp(se), _dp(up),
                                 _dp(sa), dt, inv_voxel_volume)

    @staticmethod
    def run(w, steps, with_sources=True, initial_clamp=False, field=None):
        """[diffuse_decay_step; cell_sources_sinks_step] x steps for a Workload."""
        shape = w.n
        S = w.S
        h = (w.dx, w.dx, w.dx)
        rho = w.initial_field() if field is None else _f(field).copy()
        ws = Oracle.workspaces(shape, h, w.diffusion, w.decay, w.dt)
        dv, dm, dx_ = w.dirichlet_entries()
        grouping = Oracle.group(w.agent_ids, w.agent_pos, w.bounds(), h, shape) if w.n_agents else None
        inv_vox = 1.0 / (h[0] * h[1] * h[2])
        if initial_clamp:
            Oracle.dirichlet(rho, S, dv, dm, dx_)
        for _ in range(steps):
            Oracle.sweep(rho, shape, S, 0, ws[0])
            if 1 in ws:
                Oracle.sweep(rho, shape, S, 1, ws[1])
            if 2 in ws:
                Oracle.sweep(rho, shape, S, 2, ws[2])
            Oracle.dirichlet(rho, S, dv, dm, dx_)
            if with_sources and grouping is not None:
                Oracle.sources(rho, S, grouping, w.agent_vol, w.agent_sec, w.agent_upt, w.agent_sat, w.dt, inv_vox)
        return rho


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libbiodiff_ref.so)
# --------------------------------------------------------------------------
class Reference:
    """The unmodified reference code driven through ref_shim.cpp."""

    def __init__(self, w, workers=0, staged=False, dirichlet=True, agents=True):
        L = ref_lib()
        self.w = w
        b = _f(w.bounds())
        h = _f([w.dx, w.dx, w.dx])
        h_ = _vp()
        _rchk(L.ref_create(_dp(b), _dp(h), w.S, _dp(_f(w.diffusion)), _dp(_f(w.decay)), _dp(_f(w.initial)),
                           int(workers), 1 if staged else 0, ctypes.byref(h_)))
        self.h = h_
        dims = (ctypes.c_int * 3)()
        L.ref_mesh_dims(self.h, dims)
        self.shape = tuple(dims)
        if dirichlet:
            mask, vals = w.boundary_clamp()
            if mask.any():
                _rchk(L.ref_add_boundary_dirichlet(self.h, mask.ctypes.data_as(_P(_u8)), _dp(_f(vals))))
            if w.interior_dirichlet is not None:
                iv, im, ival = w.interior_dirichlet
                iv = _i(iv)
                im = np.ascontiguousarray(im, np.uint8)
                _rchk(L.ref_add_dirichlet(self.h, iv.size, _ip(iv), im.ctypes.data_as(_P(_u8)), _dp(_f(ival))))
        if agents and w.n_agents:
            _rchk(L.ref_set_agents(self.h, w.n_agents, _ip(_i(w.agent_ids)), _dp(_f(w.agent_pos)),
                                   _dp(_f(w.agent_vol)), _dp(_f(w.agent_sec)), _dp(_f(w.agent_upt)),
                                   _dp(_f(w.agent_sat))))
        _rchk(L.ref_build_workspaces(self.h, w.dt))

    def load_agents(self, path, names):
        """load_agents (config.cpp:416-477) over the reference's text.cpp + AgentPopulation."""
        L = ref_lib()
        nm = (ctypes.c_char_p * max(1, len(names)))(*[str(x).encode() for x in names])
        _rchk(L.ref_load_agents(self.h, str(path).encode(), nm, len(names)))
        n, S = int(L.ref_agent_count(self.h)), len(names)
        ids = np.zeros(n, np.int64)
        pos, vol = np.zeros((n, 3)), np.zeros(n)
        sec, upt, sat = np.zeros((n, S)), np.zeros((n, S)), np.zeros((n, S))
        _rchk(L.ref_get_agents(self.h, _ip(ids), _dp(pos), _dp(vol), _dp(sec), _dp(upt), _dp(sat)))
        return ids, pos, vol, sec, upt, sat

    def close(self):
        if getattr(self, "h", None):
            ref_lib().ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def count(self):
        return self.shape[0] * self.shape[1] * self.shape[2] * self.w.S

    def field(self):
        out = np.empty(self.count)
        _rchk(ref_lib().ref_get_field(self.h, _dp(out), out.size))
        return out

    def field_range(self, offset, count, out):
        _rchk(ref_lib().ref_get_field_range(self.h, int(offset), int(count), _dp(out)))

    def field_digest(self) -> str:
        return field_sha256(self.field_range, self.count)

    def set_field(self, values):
        v = _f(values)
        _rchk(ref_lib().ref_set_field(self.h, _dp(v), v.size))

    def workspace(self, axis):
        n = self.shape[axis]
        S = self.w.S
        q, dinv, cb = np.zeros(S), np.zeros(n * S), np.zeros(n * S)
        dims = ctypes.c_int()
        rc = ref_lib().ref_get_workspace(self.h, axis, _dp(q), _dp(dinv), _dp(cb), ctypes.byref(dims))
        if rc == 3:
            return None
        _rchk(rc)
        return q, dinv, cb, dims.value

    def dirichlet(self):
        L = ref_lib()
        E = L.ref_dirichlet_size(self.h)
        S = self.w.S
        v = np.zeros(E, np.int64)
        m = np.zeros(E * S, np.uint8)
        x = np.zeros(E * S)
        L.ref_get_dirichlet(self.h, _ip(v), m.ctypes.data_as(_P(_u8)), _dp(x))
        return v, m.reshape(E, S), x.reshape(E, S)

    def grouping(self):
        L = ref_lib()
        G = L.ref_group_count(self.h)
        n = self.w.n_agents
        gv, go, order = np.zeros(max(G, 1), np.int64), np.zeros(G + 1, np.int64), np.zeros(max(n, 1), np.int64)
        L.ref_get_grouping(self.h, _ip(gv), _ip(go), _ip(order))
        return gv[:G], go, order[:n]

    def sweep(self, axis):
        _rchk(ref_lib().ref_sweep(self.h, axis))

    def apply_dirichlet(self):
        _rchk(ref_lib().ref_apply_dirichlet(self.h))

    def diffuse_decay_step(self):
        _rchk(ref_lib().ref_diffuse_decay_step(self.h))

    def sources(self, dt):
        _rchk(ref_lib().ref_sources_step(self.h, dt))

    def snapshot(self, table: bool, substrate: int, z_slice: int) -> str:
        """validation.cpp:155-200 snapshot text of the current field."""
        L = ref_lib()
        need = L.ref_snapshot(self.h, 1 if table else 0, substrate, z_slice, None, 0)
        if need < 0:
            raise RefError(2, L.ref_last_error().decode())
        buf = ctypes.create_string_buffer(int(need))
        L.ref_snapshot(self.h, 1 if table else 0, substrate, z_slice, buf, need)
        return buf.value.decode()

    def run(self, steps, with_sources=True):
        """Returns the steady_clock seconds of the step loop alone."""
        sec = _d()
        _rchk(ref_lib().ref_run(self.h, int(steps), self.w.dt, 1 if with_sources else 0, ctypes.byref(sec)))
        return sec.value


def ref_convergence(kind: int, levels: int):
    o, st, er, p = _d(), np.zeros(levels), np.zeros(levels), ctypes.c_int()
    _rchk(ref_lib().ref_convergence(kind, levels, ctypes.byref(o), _dp(st), _dp(er), ctypes.byref(p)))
    return o.value, st, er, bool(p.value)


def ref_format_double(v: float) -> str:
    buf = ctypes.create_string_buffer(64)
    _rchk(ref_lib().ref_format_double(v, buf, 64))
    return buf.value.decode()


def ref_cross_check(a, b, substrates: int, abs_tol: float, rel_tol: float):
    """The reference's own cross_check (validation.cpp:112-137): (max_abs, max_rel, worst index, pass)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    ma, mr, wi, p = _d(), _d(), _i64(), ctypes.c_int()
    _rchk(ref_lib().ref_cross_check(_dp(a), _dp(b), a.size, substrates, abs_tol, rel_tol, ctypes.byref(ma),
                                    ctypes.byref(mr), ctypes.byref(wi), ctypes.byref(p)))
    return ma.value, mr.value, int(wi.value), bool(p.value)


def ref_mutant_check():
    f = (ctypes.c_int * 3)()
    _rchk(ref_lib().ref_mutant_check(f))
    return tuple(bool(x) for x in f)


def time_reference(w, steps, workers, warmup=1, with_sources=True):
    """Times the reference step loop on this host; returns (seconds, steps)."""
    r = Reference(w, workers=workers)
    if warmup:
        r.run(warmup, with_sources)
    t = r.run(steps, with_sources)
    r.close()
    return t


def nproc():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def now():
    return time.perf_counter()


# ---- the reference's own XML config layer (config.cpp via oracle/boost_shim) ----

def _ref_cfg():
    L = ref_lib()
    if not getattr(L, "_cfg_bound", False):
        L.ref_config_last_error.restype = ctypes.c_char_p
        L.ref_config_canonical.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _i64, _P(_i64)]
        L.ref_config_build.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _P(_i64), _P(ctypes.c_int), _P(_i64),
                                       _P(_i64), _P(_d), _P(_i64), _P(_u8), _P(_d), _P(_i64), _P(_d), _P(_d),
                                       _P(_d), _P(_d), _P(_d)]
        L.ref_config_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, _i64, ctypes.c_int, _P(_d), _i64]
        L._cfg_bound = True
    return L


def _cfg_args(xml, path):
    return (xml.encode() if xml is not None else None), (str(path).encode() if path is not None else None)


def ref_config_canonical(xml=None, path=None):
    """(status, text): serialize_config(parse_config...) of the reference
    (config.cpp:295-398), or its error status (1 config_error, 4 io_error)
    and message."""
    L = _ref_cfg()
    x, p = _cfg_args(xml, path)
    need = _i64()
    rc = L.ref_config_canonical(x, p, None, 0, ctypes.byref(need))
    if rc:
        return rc, L.ref_config_last_error().decode()
    buf = ctypes.create_string_buffer(need.value)
    L.ref_config_canonical(x, p, buf, need.value, ctypes.byref(need))
    return 0, buf.value.decode()


def ref_config_build(xml=None, path=None):
    """build_microenvironment + build_agents of the reference (config.cpp:494-566)."""
    L = _ref_cfg()
    x, p = _cfg_args(xml, path)
    nv, S, nd, na = _i64(), ctypes.c_int(), _i64(), _i64()
    rc = L.ref_config_build(x, p, ctypes.byref(nv), ctypes.byref(S), ctypes.byref(nd), ctypes.byref(na),
                            *([None] * 10))
    if rc:
        raise RuntimeError(L.ref_config_last_error().decode())
    S_, nd_, na_ = S.value, nd.value, na.value
    out = {"S": S_, "field": np.empty(nv.value * S_), "dir_voxel": np.empty(nd_, np.int64),
           "dir_mask": np.empty(nd_ * S_, np.uint8), "dir_values": np.empty(nd_ * S_),
           "ids": np.empty(na_, np.int64), "positions": np.empty(3 * na_), "volume": np.empty(na_),
           "secretion": np.empty(na_ * S_), "uptake": np.empty(na_ * S_), "saturation": np.empty(na_ * S_)}
    types = {"dir_voxel": _i64, "dir_mask": _u8, "ids": _i64}
    ptrs = [out[k].ctypes.data_as(_P(types.get(k, _d))) for k in
            ("field", "dir_voxel", "dir_mask", "dir_values", "ids", "positions", "volume", "secretion", "uptake",
             "saturation")]
    L.ref_config_build(x, p, ctypes.byref(nv), ctypes.byref(S), ctypes.byref(nd), ctypes.byref(na), *ptrs)
    return out


def ref_config_run(steps, xml=None, path=None, workers=0, count=None):
    """The reference's step loop from a config: the final field."""
    L = _ref_cfg()
    x, p = _cfg_args(xml, path)
    if count is None:
        count = ref_config_build(xml, path)["field"].size
    field = np.empty(count)
    rc = L.ref_config_run(x, p, steps, workers, field.ctypes.data_as(_P(_d)), count)
    if rc:
        raise RuntimeError(L.ref_config_last_error().decode())
    return field
