"""B200-native LOD diffusion step (arxiv 2110.13368 hot path).

Python binding of the C ABI in ``include/biodiff_b200.h`` (ctypes over the
in-tree ``_lib/libbiodiff_b200.so``). The compute path is the CUDA library
only: importing works without a GPU (for the host helpers), but creating a
:class:`Session` needs an sm_100 device and fails loudly otherwise — there
is no CPU fallback.

The names mirror the reference's C++ API (/root/reference/proj/src/core):
``diffuse_decay_step`` (solver.hpp:72), ``cell_sources_sinks_step``
(agents.hpp:72), ``diffusion_sweep`` (solver.hpp:51),
``apply_dirichlet_conditions`` (solver.hpp:55),
``precompute_thomas_coefficients`` (solver.hpp:38), ``cross_check``
(validation.hpp:64), with errors raised as the reference's exception
categories (errors.hpp:9-24).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = [
    "LIB_PATH", "lib", "BiodiffError", "ConfigError", "StateError", "IOError_",
    "Mesh", "Session", "mesh_from_bounds", "nearest_voxel", "precompute_thomas_coefficients",
    "device_count", "AXIS_X", "AXIS_Y", "AXIS_Z", "KERNEL_CLASSES",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", os.environ.get("BIODIFF_LIB", "libbiodiff_b200.so"))

AXIS_X, AXIS_Y, AXIS_Z = 0, 1, 2
KERNEL_CLASSES = ("sweep_x", "sweep_y", "sweep_z", "dirichlet", "sources", "aux", "sweep_xy", "sweep_xyz",
                  "resident")


class BiodiffError(RuntimeError):
    code = 2


class ConfigError(BiodiffError):
    """config_error (errors.hpp:9-12), status 1."""
    code = 1


class StateError(BiodiffError):
    """state_error / argument / domain / CUDA errors (errors.hpp:19-22), status 2."""
    code = 2


class IOError_(BiodiffError):
    """io_error (errors.hpp:14-17), status 4."""
    code = 4


class Mesh(ctypes.Structure):
    """CartesianMesh (mesh.hpp:17-57) as the C ABI's biodiff_mesh."""

    _fields_ = [
        ("x_min", ctypes.c_double), ("x_max", ctypes.c_double),
        ("y_min", ctypes.c_double), ("y_max", ctypes.c_double),
        ("z_min", ctypes.c_double), ("z_max", ctypes.c_double),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
    ]

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def voxel_count(self) -> int:
        return int(self.nx) * int(self.ny) * int(self.nz)

    @property
    def voxel_volume(self) -> float:
        return self.dx * self.dy * self.dz

    def bounds(self):
        return (self.x_min, self.x_max, self.y_min, self.y_max, self.z_min, self.z_max)

    def __repr__(self):
        return f"Mesh({self.nx}x{self.ny}x{self.nz}, h=({self.dx},{self.dy},{self.dz}))"


_P = ctypes.POINTER
_d = ctypes.c_double
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
# biodiff_plane_exchange (include/biodiff_b200.h)
PLANE_EXCHANGE = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _P(_d), _i32, _P(_d), _i32, _i64)

_SIGNATURES = {
    "biodiff_last_error": (ctypes.c_char_p, []),
    "biodiff_version": (_i32, []),
    "biodiff_build_flags": (_i32, []),
    "biodiff_config_canonical": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _i64, _P(_i64)]),
    "biodiff_config_save": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]),
    "biodiff_config_build": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _P(_i64), _P(_i32), _P(_i64), _P(_i64),
                                            _P(_d), _P(_i64), _P(ctypes.c_uint8), _P(_d), _P(_i64), _P(_d), _P(_d),
                                            _P(_d), _P(_d), _P(_d)]),
    "biodiff_session_from_config": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _i32, _P(_vp), _vp]),
    "biodiff_mesh_from_bounds": (ctypes.c_int, [_d] * 9 + [_P(Mesh)]),
    "biodiff_nearest_voxel": (ctypes.c_int, [_P(Mesh), _P(_d), _P(_i64)]),
    "biodiff_precompute_thomas": (ctypes.c_int, [_P(Mesh), _i32, _P(_d), _P(_d), _d, _i32, _i32, _P(_d), _P(_d), _P(_d)]),
    "biodiff_device_count": (ctypes.c_int, [_P(_i32)]),
    "biodiff_session_create": (ctypes.c_int, [_P(Mesh), _i32, _i32, _P(_vp)]),
    "biodiff_session_destroy": (ctypes.c_int, [_vp]),
    "biodiff_set_substrates": (ctypes.c_int, [_vp, _P(_d), _P(_d), _d]),
    "biodiff_set_workspace": (ctypes.c_int, [_vp, _i32, _i32, _i32, _d, _P(_d), _P(_d), _P(_d)]),
    "biodiff_set_dirichlet": (ctypes.c_int, [_vp, _i64, _P(_i64), _P(ctypes.c_uint8), _P(_d)]),
    "biodiff_set_agents": (ctypes.c_int, [_vp, _i64, _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d), _P(_d)]),
    "biodiff_agent_grouping": (ctypes.c_int, [_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64)]),
    "biodiff_agent_count": (ctypes.c_int, [_vp, _P(_i64)]),
    "biodiff_set_agent_positions": (ctypes.c_int, [_vp, _P(_d), _i64]),
    "biodiff_sample_agent_densities": (ctypes.c_int, [_vp, _P(_d), _i64]),
    "biodiff_set_agent_position": (ctypes.c_int, [_vp, _i64, _P(_d)]),
    "biodiff_agent_positions_device": (ctypes.c_int, [_vp, _P(_vp)]),
    "biodiff_rebuild_voxel_grouping": (ctypes.c_int, [_vp]),
    "biodiff_download_agents": (ctypes.c_int, [_vp, _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d), _P(_d)]),
    "biodiff_load_agents_csv": (ctypes.c_int, [_vp, ctypes.c_char_p, _P(ctypes.c_char_p)]),
    "biodiff_save_agents_csv": (ctypes.c_int, [_vp, ctypes.c_char_p, _P(ctypes.c_char_p)]),
    "biodiff_parse_agents_csv": (ctypes.c_int, [_P(Mesh), ctypes.c_char_p, _P(ctypes.c_char_p), _i32, _P(_i64),
                                                _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d), _P(_d)]),
    "biodiff_write_agents_csv": (ctypes.c_int, [ctypes.c_char_p, _P(ctypes.c_char_p), _i32, _i64, _P(_i64), _P(_d),
                                                _P(_d), _P(_d), _P(_d), _P(_d)]),
    "biodiff_upload_field": (ctypes.c_int, [_vp, _P(_d), _i64]),
    # engine (typed bindings with the clock / metrics structs: engine.py)
    "biodiff_clock_make": (ctypes.c_int, [_d, _d, _d, _d, _vp]),
    "biodiff_run_simulation": (ctypes.c_int, [_vp, _vp, _i32, _d, _vp, _vp, _vp, _vp, _vp]),
    "biodiff_translate_vector_to_array": (ctypes.c_int, [_P(_P(_d)), _P(_i64), _i64, _P(_d), _P(_i32)]),
    "biodiff_upload_field_nested": (ctypes.c_int, [_vp, _P(_P(_d)), _P(_i64), _i64]),
    "biodiff_download_field_nested": (ctypes.c_int, [_vp, _P(_P(_d)), _i64]),
    "biodiff_field_all_finite": (ctypes.c_int, [_vp, _P(_i32)]),
    "biodiff_fill_field": (ctypes.c_int, [_vp, _P(_d)]),
    "biodiff_download_field": (ctypes.c_int, [_vp, _P(_d), _i64]),
    "biodiff_download_field_range": (ctypes.c_int, [_vp, _i64, _i64, _P(_d)]),
    "biodiff_diffusion_sweep": (ctypes.c_int, [_vp, _i32]),
    "biodiff_apply_dirichlet": (ctypes.c_int, [_vp]),
    "biodiff_diffuse_decay_step": (ctypes.c_int, [_vp]),
    "biodiff_cell_sources_sinks_step": (ctypes.c_int, [_vp, _d]),
    "biodiff_shard_create": (ctypes.c_int, [_P(Mesh), _i32, _i32, _i32, _i32, _i32, _i32, _P(_vp)]),
    "biodiff_shard_info": (ctypes.c_int, [_vp, _P(_i32), _P(_i32), _P(_i32)]),
    "biodiff_upload_field_global": (ctypes.c_int, [_vp, _P(_d), _i64]),
    "biodiff_download_field_global": (ctypes.c_int, [_vp, _P(_d), _i64]),
    "biodiff_zslab_connect_host": (ctypes.c_int, [_vp, _i32, _i32, PLANE_EXCHANGE, _vp]),
    "biodiff_advance": (ctypes.c_int, [_vp, _i64, _d, _i32]),
    "biodiff_prepare_advance": (ctypes.c_int, [_vp, _i64, _d, _i32]),
    "biodiff_synchronize": (ctypes.c_int, [_vp]),
    "biodiff_session_stream": (ctypes.c_int, [_vp, _P(_vp)]),
    "biodiff_set_kernel_timing": (ctypes.c_int, [_vp, _i32]),
    "biodiff_kernel_times": (ctypes.c_int, [_vp, _P(_i32), _P(_i64), _P(_d)]),
    "biodiff_event_record": (ctypes.c_int, [_vp, _i32]),
    "biodiff_event_elapsed": (ctypes.c_int, [_vp, _i32, _i32, _P(_d)]),
    "biodiff_launch_count": (ctypes.c_int, [_vp, _P(_i64)]),
    "biodiff_cross_check": (ctypes.c_int, [_vp, _P(_d), _i64, _d, _d, _P(_d), _P(_d), _P(_i64), _P(_i32)]),
    "biodiff_ensemble_create": (ctypes.c_int, [_P(Mesh), _i32, _i32, _i32, _P(_vp)]),
    "biodiff_ensemble_set_substrates": (ctypes.c_int, [_vp, _P(_d), _P(_d), _d]),
    "biodiff_ensemble_set_agents": (ctypes.c_int, [_vp, _i64, _P(_i32), _P(_i64), _P(_d), _P(_d), _P(_d), _P(_d),
                                                   _P(_d)]),
    "biodiff_zslab_create": (ctypes.c_int, [_P(Mesh), _i32, _i32, _i32, _i32, _P(_vp)]),
    "biodiff_zslab_info": (ctypes.c_int, [_vp, _P(_i32), _P(_i32), _P(_i32)]),
    "biodiff_nccl_unique_id": (ctypes.c_int, [_P(ctypes.c_uint8)]),
    "biodiff_zslab_connect_nccl": (ctypes.c_int, [_vp, _P(ctypes.c_uint8), _i32, _i32]),
    "biodiff_zslab_link_local": (ctypes.c_int, [_P(_vp), _i32]),
    "biodiff_zslab_group_advance": (ctypes.c_int, [_P(_vp), _i32, _i64, _d, _i32]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Loads the in-tree CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2110_13368_b200` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _check(status: int):
    if status == 0:
        return
    msg = lib().biodiff_last_error().decode(errors="replace")
    cls = {1: ConfigError, 2: StateError, 4: IOError_}.get(status, BiodiffError)
    raise cls(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_P(_d))


def _f64(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a


def mesh_from_bounds(x_min, x_max, y_min, y_max, z_min, z_max, dx, dy, dz) -> Mesh:
    """CartesianMesh::from_bounds (mesh.cpp:12-44)."""
    m = Mesh()
    _check(lib().biodiff_mesh_from_bounds(x_min, x_max, y_min, y_max, z_min, z_max, dx, dy, dz, ctypes.byref(m)))
    return m


def nearest_voxel(mesh: Mesh, position) -> int:
    """CartesianMesh::nearest_voxel (mesh.cpp:72-88)."""
    p = _f64(position, 3)
    out = _i64()
    _check(lib().biodiff_nearest_voxel(ctypes.byref(mesh), _dptr(p), ctypes.byref(out)))
    return int(out.value)


def translate_vector_to_array(nested):
    """translate_vector_to_array (mesh.cpp:101-119) on the host: (flat values, substrate count)."""
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in nested]
    ptrs = (_P(_d) * max(1, len(arrs)))(*[_dptr(a) for a in arrs])
    counts = np.array([a.size for a in arrs] or [0], dtype=np.int64)
    S = _i32()
    _check(lib().biodiff_translate_vector_to_array(ptrs, counts.ctypes.data_as(_P(_i64)), len(arrs), None,
                                                   ctypes.byref(S)))
    out = np.empty(len(arrs) * S.value)
    _check(lib().biodiff_translate_vector_to_array(ptrs, counts.ctypes.data_as(_P(_i64)), len(arrs), _dptr(out),
                                                   ctypes.byref(S)))
    return out, int(S.value)


def parse_agents_csv(mesh: Mesh, path: str, names):
    """load_agents (config.cpp:416-477) on the host: parse + validate an agent file.
    Returns (ids, xyz[n,3], volume, secretion[n,S], uptake[n,S], saturation[n,S])."""
    S = len(names)
    nm = (ctypes.c_char_p * max(1, S))(*[str(x).encode() for x in names])
    n = _i64()
    p = str(path).encode()
    _check(lib().biodiff_parse_agents_csv(ctypes.byref(mesh), p, nm, S, ctypes.byref(n), None, None, None, None,
                                          None, None))
    N = int(n.value)
    ids = np.zeros(N, np.int64)
    xyz, vol = np.zeros((N, 3)), np.zeros(N)
    sec, upt, sat = np.zeros((N, S)), np.zeros((N, S)), np.zeros((N, S))
    _check(lib().biodiff_parse_agents_csv(ctypes.byref(mesh), p, nm, S, ctypes.byref(n), ids.ctypes.data_as(_P(_i64)),
                                          _dptr(xyz), _dptr(vol), _dptr(sec), _dptr(upt), _dptr(sat)))
    return ids, xyz, vol, sec, upt, sat


def write_agents_csv(path: str, names, ids, xyz, volume, secretion, uptake, saturation):
    """save_agents (config.cpp:479-491): the reference's agent file format."""
    S = len(names)
    nm = (ctypes.c_char_p * max(1, S))(*[str(x).encode() for x in names])
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64).ravel())
    n = ids.size
    _check(lib().biodiff_write_agents_csv(str(path).encode(), nm, S, n, ids.ctypes.data_as(_P(_i64)),
                                          _dptr(_f64(xyz, 3 * n)), _dptr(_f64(volume, n)),
                                          _dptr(_f64(secretion, n * S)), _dptr(_f64(uptake, n * S)),
                                          _dptr(_f64(saturation, n * S))))


def precompute_thomas_coefficients(mesh: Mesh, diffusion, decay, dt: float, axis: int, dims: int):
    """precompute_thomas_coefficients (solver.cpp:47-97) -> (off_diag[S], denom_inv[n,S], c_back[n,S])."""
    D = _f64(diffusion)
    L = _f64(decay, D.size)
    S = D.size
    n = (mesh.nx, mesh.ny, mesh.nz)[axis]
    q = np.zeros(S)
    dinv = np.zeros(n * S)
    cb = np.zeros(n * S)
    _check(lib().biodiff_precompute_thomas(ctypes.byref(mesh), S, _dptr(D), _dptr(L), dt, axis, dims,
                                           _dptr(q), _dptr(dinv), _dptr(cb)))
    return q, dinv.reshape(n, S), cb.reshape(n, S)


def _cfg_args(xml, path):
    if (xml is None) == (path is None):
        raise ValueError("give exactly one of xml (a document) or path (a file)")
    return (xml.encode() if xml is not None else None), (str(path).encode() if path is not None else None)


def config_canonical(xml: Optional[str] = None, path=None) -> str:
    """serialize_config(parse_config...) of an XML configuration (the
    reference's schema, config.hpp:75-91): the canonical document."""
    x, p = _cfg_args(xml, path)
    need = _i64()
    _check(lib().biodiff_config_canonical(x, p, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().biodiff_config_canonical(x, p, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def config_save(out_path, xml: Optional[str] = None, path=None) -> None:
    """save_config: writes the canonical document of a configuration."""
    x, p = _cfg_args(xml, path)
    _check(lib().biodiff_config_save(x, p, str(out_path).encode()))


def config_build(xml: Optional[str] = None, path=None) -> dict:
    """build_microenvironment + build_agents of a configuration (config.cpp:494-566):
    the initial field, the Dirichlet entries and the agents, as arrays."""
    x, p = _cfg_args(xml, path)
    nv, S, nd, na = _i64(), _i32(), _i64(), _i64()
    nul = [None] * 10
    _check(lib().biodiff_config_build(x, p, ctypes.byref(nv), ctypes.byref(S), ctypes.byref(nd), ctypes.byref(na),
                                      *nul))
    S_, nd_, na_ = int(S.value), int(nd.value), int(na.value)
    out = {"S": S_, "field": np.empty(int(nv.value) * S_), "dir_voxel": np.empty(nd_, np.int64),
           "dir_mask": np.empty(nd_ * S_, np.uint8), "dir_values": np.empty(nd_ * S_), "ids": np.empty(na_, np.int64),
           "positions": np.empty(3 * na_), "volume": np.empty(na_), "secretion": np.empty(na_ * S_),
           "uptake": np.empty(na_ * S_), "saturation": np.empty(na_ * S_)}
    ptrs = [out[k].ctypes.data_as(_P(t)) for k, t in (("field", _d), ("dir_voxel", _i64), ("dir_mask", ctypes.c_uint8),
                                                      ("dir_values", _d), ("ids", _i64), ("positions", _d),
                                                      ("volume", _d), ("secretion", _d), ("uptake", _d),
                                                      ("saturation", _d))]
    _check(lib().biodiff_config_build(x, p, ctypes.byref(nv), ctypes.byref(S), ctypes.byref(nd), ctypes.byref(na),
                                      *ptrs))
    return out


def session_from_config(xml: Optional[str] = None, path=None, device: int = 0):
    """A ready Session for a configuration (mesh, coefficients at dt_diff,
    boundary Dirichlet shell, agents, initial field) and its clock
    (dt_diff, dt_mech, dt_cell, max_time, total_steps)."""
    import re
    from paper_2110_13368_b200.engine import CClock
    x, p = _cfg_args(xml, path)
    h = _vp()
    clk = CClock()
    _check(lib().biodiff_session_from_config(x, p, device, ctypes.byref(h), ctypes.addressof(clk)))
    canon = config_canonical(xml=xml, path=path)
    num = {k: float(v) for k, v in re.findall(r"<(x_min|x_max|y_min|y_max|z_min|z_max|dx|dy|dz)>([^<]+)<", canon)}
    mesh = mesh_from_bounds(num["x_min"], num["x_max"], num["y_min"], num["y_max"], num["z_min"], num["z_max"],
                            num["dx"], num["dy"], num["dz"])
    s = Session.__new__(Session)
    s.mesh, s.S_total, s.S = mesh, canon.count("<substrate>"), canon.count("<substrate>")
    s.zslab, s.shard, s.replicas = None, None, 1
    s._h = h
    clock = {k: getattr(clk, k) for k in ("dt_diff", "dt_mech", "dt_cell", "t_max", "per_mech", "per_cell",
                                          "total_steps")}
    return s, clock


def experimental_build() -> bool:
    """True when the library was built with EXPERIMENTAL=1 (the measured-and-
    rejected kernel variants compiled in for A/B runs)."""
    return bool(lib().biodiff_build_flags() & 1)


def device_count() -> int:
    n = _i32()
    _check(lib().biodiff_device_count(ctypes.byref(n)))
    return int(n.value)


@dataclass
class CrossCheckReport:
    """validation.hpp:52-59."""
    max_abs: float
    max_rel: float
    worst_value_index: int
    worst_voxel: int
    worst_substrate: int
    passed: bool


class Session:
    """A device-resident Microenvironment plus the execution strategy that
    replaces WorkerPool& (backend.hpp:34). Mirrors the reference entry
    points; the field stays on the device until :meth:`download_field`."""

    def __init__(self, mesh: Mesh, substrates: int, device: int = 0, zslab=None, replicas: int = 1, shard=None):
        """zslab=(z0, z1): a z-slab session owning global planes [z0, z1) of
        `mesh` (the global mesh); its field holds only those planes.
        shard=(s0, s1): a substrate shard holding substrates [s0, s1) of the
        `substrates`-substrate problem (combinable with zslab). Parameter
        arrays (set_substrates, set_dirichlet, set_agents, fill_field) are
        GLOBAL ([substrates] columns); field buffers are the session's own
        layout (``S`` = s1 - s0 values per voxel), or GLOBAL through
        upload_field_global / download_field_global.
        replicas > 1: an ensemble of independent microenvironments stacked
        replica-major (values[(r*voxels + v)*S + s])."""
        self.mesh = mesh
        self.S_total = int(substrates)
        self.S = int(substrates)
        self.zslab = None
        self.shard = None
        self.replicas = int(replicas)
        h = _vp()
        if self.replicas > 1:
            _check(lib().biodiff_ensemble_create(ctypes.byref(mesh), self.S, self.replicas, device, ctypes.byref(h)))
        elif shard is not None:
            s0, s1 = (int(x) for x in shard)
            z0, z1 = (int(z) for z in zslab) if zslab is not None else (0, int(mesh.nz))
            _check(lib().biodiff_shard_create(ctypes.byref(mesh), self.S_total, s0, s1, z0, z1, device,
                                              ctypes.byref(h)))
            self.shard = (s0, s1)
            self.S = s1 - s0
            if (z0, z1) != (0, int(mesh.nz)):
                self.zslab = (z0, z1)
        elif zslab is None:
            _check(lib().biodiff_session_create(ctypes.byref(mesh), self.S, device, ctypes.byref(h)))
        else:
            z0, z1 = (int(z) for z in zslab)
            _check(lib().biodiff_zslab_create(ctypes.byref(mesh), self.S, z0, z1, device, ctypes.byref(h)))
            self.zslab = (z0, z1)
        self._h = h

    # -- z-slab transports ---------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().biodiff_nccl_unique_id(buf))
        return bytes(buf)

    def connect_host_transport(self, nranks: int, rank: int, exchange):
        """One slab per process with the planes moved by `exchange(send, send_peer,
        recv, recv_peer)` (numpy views of the pinned staging planes, or None):
        send `send` to rank send_peer, fill `recv` from recv_peer (e.g. gloo)."""
        def cb(_user, send, send_peer, recv, recv_peer, count):
            try:
                sv = np.ctypeslib.as_array(send, (count,)) if send else None
                rv = np.ctypeslib.as_array(recv, (count,)) if recv else None
                exchange(sv, int(send_peer), rv, int(recv_peer))
                return 0
            except BaseException as e:  # surfaced by the failing call
                self._xchg_error = e
                return 1
        self._xchg_cb = PLANE_EXCHANGE(cb)  # keep alive as long as the session
        _check(lib().biodiff_zslab_connect_host(self._h, nranks, rank, self._xchg_cb, None))

    def connect_nccl(self, unique_id: bytes, nranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().biodiff_zslab_connect_nccl(self._h, buf, nranks, rank))

    @staticmethod
    def link_local(sessions):
        arr = (_vp * len(sessions))(*[s._h for s in sessions])
        _check(lib().biodiff_zslab_link_local(arr, len(sessions)))

    @staticmethod
    def group_advance(sessions, steps: int, dt: float, with_sources: bool = True):
        arr = (_vp * len(sessions))(*[s._h for s in sessions])
        _check(lib().biodiff_zslab_group_advance(arr, len(sessions), int(steps), dt, 1 if with_sources else 0))

    # -- lifetime -------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().biodiff_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def value_count(self) -> int:
        if self.zslab is not None:
            return int(self.mesh.nx) * int(self.mesh.ny) * (self.zslab[1] - self.zslab[0]) * self.S
        return self.mesh.voxel_count * self.S * self.replicas

    # -- ensembles ---------------------------------------------------------
    def ensemble_set_substrates(self, diffusion, decay, dt: float):
        """Per-replica SolverWorkspaces::build: diffusion/decay shaped [replicas, S]."""
        n = self.replicas * self.S
        _check(lib().biodiff_ensemble_set_substrates(self._h, _dptr(_f64(diffusion, n)), _dptr(_f64(decay, n)), dt))

    def ensemble_set_agents(self, replica, ids, positions, volume, secretion, uptake, saturation):
        rep = np.ascontiguousarray(np.asarray(replica, dtype=np.int32).ravel())
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64).ravel())
        n = ids.size
        _check(lib().biodiff_ensemble_set_agents(
            self._h, n, rep.ctypes.data_as(_P(_i32)), ids.ctypes.data_as(_P(_i64)), _dptr(_f64(positions, 3 * n)),
            _dptr(_f64(volume, n)), _dptr(_f64(secretion, n * self.S)), _dptr(_f64(uptake, n * self.S)),
            _dptr(_f64(saturation, n * self.S))))

    # -- set-up ---------------------------------------------------------
    def set_substrates(self, diffusion, decay, dt: float):
        """SolverWorkspaces::build (solver.cpp:277-287) + upload."""
        _check(lib().biodiff_set_substrates(self._h, _dptr(_f64(diffusion, self.S_total)),
                                            _dptr(_f64(decay, self.S_total)), dt))

    def set_workspace(self, axis: int, dims: int, dt: float, off_diag, denom_inv, c_back):
        n = (self.mesh.nx, self.mesh.ny, self.mesh.nz)[axis]
        _check(lib().biodiff_set_workspace(self._h, axis, n, dims, dt, _dptr(_f64(off_diag, self.S)),
                                           _dptr(_f64(denom_inv, n * self.S)), _dptr(_f64(c_back, n * self.S))))

    def set_dirichlet(self, voxels, mask, values):
        """DirichletMap entries (mesh.hpp:113-141); add-merge semantics."""
        v = np.ascontiguousarray(np.asarray(voxels, dtype=np.int64).ravel())
        m = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8).reshape(v.size * self.S_total))
        x = _f64(values, v.size * self.S_total)
        _check(lib().biodiff_set_dirichlet(self._h, v.size, v.ctypes.data_as(_P(_i64)),
                                           m.ctypes.data_as(_P(ctypes.c_uint8)), _dptr(x)))

    def set_agents(self, ids, positions, volume, secretion, uptake, saturation):
        """AgentPopulation (agents.cpp:12-73): host validation, device (voxel, id) grouping (csrc/agents.cu)."""
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64).ravel())
        n = ids.size
        _check(lib().biodiff_set_agents(
            self._h, n, ids.ctypes.data_as(_P(_i64)), _dptr(_f64(positions, 3 * n)), _dptr(_f64(volume, n)),
            _dptr(_f64(secretion, n * self.S_total)), _dptr(_f64(uptake, n * self.S_total)),
            _dptr(_f64(saturation, n * self.S_total))))

    def agent_grouping(self):
        g = _i64()
        _check(lib().biodiff_agent_grouping(self._h, ctypes.byref(g), None, None, None))
        G = int(g.value)
        gv = np.zeros(G, np.int64)
        go = np.zeros(G + 1, np.int64)
        # order length = total agents = go[-1]; query with a generous buffer first
        order = np.zeros(max(1, self._agent_capacity(G)), np.int64)
        _check(lib().biodiff_agent_grouping(self._h, ctypes.byref(g), gv.ctypes.data_as(_P(_i64)),
                                            go.ctypes.data_as(_P(_i64)), order.ctypes.data_as(_P(_i64))))
        return gv, go, order[: go[-1]]

    def _agent_capacity(self, G):
        return self.agent_count()

    # -- moving agents / agent files ------------------
    def agent_count(self) -> int:
        n = _i64()
        _check(lib().biodiff_agent_count(self._h, ctypes.byref(n)))
        return int(n.value)

    def set_agent_positions(self, xyz):
        """Every agent's position (agent-index order); the grouping is stale until rebuilt."""
        n = self.agent_count()
        _check(lib().biodiff_set_agent_positions(self._h, _dptr(_f64(xyz, 3 * n)), n))

    def set_agent_position(self, agent_id: int, xyz):
        """AgentPopulation::set_position (agents.cpp:45-54)."""
        _check(lib().biodiff_set_agent_position(self._h, int(agent_id), _dptr(_f64(xyz, 3))))

    def agent_positions_device(self) -> int:
        """Device address of the xyz[3n] position buffer (for GPU-side movers)."""
        p = _vp()
        _check(lib().biodiff_agent_positions_device(self._h, ctypes.byref(p)))
        return int(p.value or 0)

    def rebuild_voxel_grouping(self):
        """AgentPopulation::rebuild_voxel_grouping (agents.cpp:56-73), on the device."""
        _check(lib().biodiff_rebuild_voxel_grouping(self._h))

    def sample_agent_densities(self, out=None):
        """Densities at every agent's voxel (after the last rebuild) as [n, S], agent-index
        order; agents outside this session's voxels read NaN. `out` may be a
        preallocated (pinned) float64 buffer of n*S values."""
        n, S = self.agent_count(), self.S
        if out is None:
            out = np.empty((n, S))
        _check(lib().biodiff_sample_agent_densities(self._h, _dptr(out), n * S))
        return out

    def download_agents(self):
        """(ids, xyz[n,3], volume, secretion[n,S], uptake[n,S], saturation[n,S]) in agent-index order."""
        n, S = self.agent_count(), self.S
        ids = np.zeros(n, np.int64)
        xyz, vol = np.zeros((n, 3)), np.zeros(n)
        sec, upt, sat = np.zeros((n, S)), np.zeros((n, S)), np.zeros((n, S))
        _check(lib().biodiff_download_agents(self._h, ids.ctypes.data_as(_P(_i64)), _dptr(xyz), _dptr(vol),
                                             _dptr(sec), _dptr(upt), _dptr(sat)))
        return ids, xyz, vol, sec, upt, sat

    @staticmethod
    def _names(names):
        return (ctypes.c_char_p * len(names))(*[str(x).encode() for x in names])

    def load_agents_csv(self, path: str, names):
        """load_agents (config.cpp:416-477) + set_agents."""
        if len(names) != self.S_total:
            raise ValueError("one name per substrate")
        _check(lib().biodiff_load_agents_csv(self._h, str(path).encode(), self._names(names)))

    def save_agents_csv(self, path: str, names):
        """save_agents (config.cpp:479-491) of the device's current agents."""
        if len(names) != self.S_total:
            raise ValueError("one name per substrate")
        _check(lib().biodiff_save_agents_csv(self._h, str(path).encode(), self._names(names)))

    # -- field ----------------------------------------------------------
    def upload_field(self, values):
        a = _f64(values, self.value_count)
        _check(lib().biodiff_upload_field(self._h, _dptr(a), a.size))

    def upload_field_nested(self, nested):
        """PhysiCell's vector-of-vectors density (one array per voxel) -> HBM (mesh.cpp:101-119 checks)."""
        arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in nested]
        ptrs = (_P(_d) * max(1, len(arrs)))(*[_dptr(a) for a in arrs])
        counts = np.array([a.size for a in arrs], dtype=np.int64)
        _check(lib().biodiff_upload_field_nested(self._h, ptrs, counts.ctypes.data_as(_P(_i64)), len(arrs)))

    def download_field_nested(self):
        """HBM -> a list of per-voxel arrays (translate_array_to_vector, mesh.cpp:121-136)."""
        nvox = self.value_count // self.S
        arrs = [np.empty(self.S) for _ in range(nvox)]
        ptrs = (_P(_d) * max(1, nvox))(*[_dptr(a) for a in arrs])
        _check(lib().biodiff_download_field_nested(self._h, ptrs, nvox))
        return arrs

    def all_finite(self) -> bool:
        """DensityField::all_finite (mesh.cpp:95-99) on the device field."""
        f = _i32()
        _check(lib().biodiff_field_all_finite(self._h, ctypes.byref(f)))
        return bool(f.value)

    def fill_field(self, initial):
        """Every voxel := initial[S] (Microenvironment::create's initial condition)."""
        _check(lib().biodiff_fill_field(self._h, _dptr(_f64(initial, self.S_total))))

    def upload_field_global(self, values):
        """This session's planes / substrate columns of a GLOBAL a1-layout field."""
        a = _f64(values, self.mesh.voxel_count * self.S_total)
        _check(lib().biodiff_upload_field_global(self._h, _dptr(a), a.size))

    def download_field_global(self, out: np.ndarray) -> np.ndarray:
        """Writes this session's planes / substrate columns into a GLOBAL a1-layout field."""
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != self.mesh.voxel_count * self.S_total:
            raise ValueError("out must be a contiguous float64 global field")
        _check(lib().biodiff_download_field_global(self._h, _dptr(out), out.size))
        return out

    def download_field(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.value_count, np.float64)
        _check(lib().biodiff_download_field(self._h, _dptr(out), out.size))
        return out

    def download_field_range(self, offset: int, count: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """values[offset, offset + count) of the device field (download_field's flat array)."""
        if out is None:
            out = np.empty(count, np.float64)
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size < count:
            raise ValueError("out must be a contiguous float64 array of at least `count` values")
        _check(lib().biodiff_download_field_range(self._h, int(offset), int(count), _dptr(out)))
        return out[:count]

    # -- the hot path ---------------------------------------------------
    def diffusion_sweep(self, axis: int):
        _check(lib().biodiff_diffusion_sweep(self._h, axis))

    def apply_dirichlet_conditions(self):
        _check(lib().biodiff_apply_dirichlet(self._h))

    def diffuse_decay_step(self):
        _check(lib().biodiff_diffuse_decay_step(self._h))

    def cell_sources_sinks_step(self, dt: float):
        _check(lib().biodiff_cell_sources_sinks_step(self._h, dt))

    def advance(self, steps: int, dt: float, with_sources: bool = True):
        rc = lib().biodiff_advance(self._h, int(steps), dt, 1 if with_sources else 0)
        err = getattr(self, "_xchg_error", None)
        if rc != 0 and err is not None:  # a host-transport callback failed: its exception
            self._xchg_error = None
            raise err
        _check(rc)

    def prepare_advance(self, steps: int, dt: float, with_sources: bool = True):
        """Instantiates the graphs advance(steps, ...) replays, running nothing."""
        _check(lib().biodiff_prepare_advance(self._h, int(steps), dt, 1 if with_sources else 0))

    def synchronize(self):
        _check(lib().biodiff_synchronize(self._h))

    def stream(self) -> int:
        s = _vp()
        _check(lib().biodiff_session_stream(self._h, ctypes.byref(s)))
        return int(s.value or 0)

    # -- instrumentation ------------------------------------------------
    def set_kernel_timing(self, enabled: bool):
        _check(lib().biodiff_set_kernel_timing(self._h, 1 if enabled else 0))

    def kernel_times(self):
        n = _i32()
        _check(lib().biodiff_kernel_times(self._h, ctypes.byref(n), None, None))
        launches = np.zeros(n.value, np.int64)
        ms = np.zeros(n.value, np.float64)
        _check(lib().biodiff_kernel_times(self._h, ctypes.byref(n), launches.ctypes.data_as(_P(_i64)), _dptr(ms)))
        return {KERNEL_CLASSES[c]: (int(launches[c]), float(ms[c])) for c in range(n.value)}

    def event_record(self, slot: int):
        _check(lib().biodiff_event_record(self._h, slot))

    def event_elapsed(self, begin: int, end: int) -> float:
        ms = _d()
        _check(lib().biodiff_event_elapsed(self._h, begin, end, ctypes.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = _i64()
        _check(lib().biodiff_launch_count(self._h, ctypes.byref(n)))
        return int(n.value)

    def cross_check(self, other, abs_tol: float, rel_tol: float) -> CrossCheckReport:
        """Device-side cross_check of the session field against `other` (validation.cpp:112-137)."""
        b = _f64(other, self.value_count)
        ma, mr, wi, ok = _d(), _d(), _i64(), _i32()
        _check(lib().biodiff_cross_check(self._h, _dptr(b), b.size, abs_tol, rel_tol, ctypes.byref(ma),
                                         ctypes.byref(mr), ctypes.byref(wi), ctypes.byref(ok)))
        w = int(wi.value)
        return CrossCheckReport(ma.value, mr.value, w, w // self.S if w >= 0 else -1,
                                w % self.S if w >= 0 else -1, bool(ok.value))
