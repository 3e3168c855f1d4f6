"""Agent files: the library's host-side reader/writer
(csrc/host.cpp load_agents / save_agents, config.cpp:416-491) against the
reference's own pieces — text.cpp's trim / split_csv_line / parse_* /
format_* and the AgentPopulation ctor (agents.cpp:12-43), composed in
oracle/ref_shim.cpp exactly as config.cpp composes them. CPU only (no device):
bitwise-equal agents and identical error categories and messages."""
import os

import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import Reference, RefError, reference_available, ref_lib
from paper_2110_13368_b200 import workloads as W

NAMES = ["oxygen", "factor"]


def _mesh(w):
    return B.mesh_from_bounds(*w.bounds(), w.dx, w.dx, w.dx)


def _ref(w):
    return Reference(w, dirichlet=False, agents=False)


def _random_agents(rng, w, n):
    lo, hi = np.array(w.bounds()[0::2]), np.array(w.bounds()[1::2])
    ids = rng.permutation(10 * n)[:n].astype(np.int64) - 3 * n  # negative ids too
    pos = lo + rng.random((n, 3)) * (hi - lo)
    pos[: n // 10] = np.where(rng.random((n // 10, 3)) < 0.5, lo, hi)  # exactly on the faces
    vol = rng.random(n) * 3000 + 1e-300
    sec = rng.random((n, 2)) * 10 ** rng.integers(-320, 3, (n, 2)).astype(float)
    upt = rng.random((n, 2)) * 10.0
    sat = rng.random((n, 2)) * 40.0
    sec[0, 0] = 5e-324  # smallest subnormal
    upt[1, 1] = 0.0
    return ids, pos, vol, sec, upt, sat


def test_write_parse_round_trip_bitwise(tmp_path):
    rng = np.random.default_rng(11)
    w = W.make("t", (20, 16, 12), 2, 0, 1)
    a = _random_agents(rng, w, 500)
    p = tmp_path / "agents.csv"
    B.write_agents_csv(p, NAMES, *a)
    b = B.parse_agents_csv(_mesh(w), p, NAMES)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.int64), np.asarray(y).view(np.int64))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_written_bytes_match_reference_formatting(tmp_path):
    """save_agents (config.cpp:479-491): format_int / format_double (text.cpp)."""
    rng = np.random.default_rng(12)
    w = W.make("t", (10, 10, 10), 2, 0, 1)
    ids, pos, vol, sec, upt, sat = _random_agents(rng, w, 60)
    p = tmp_path / "a.csv"
    B.write_agents_csv(p, NAMES, ids, pos, vol, sec, upt, sat)
    L = ref_lib()
    import ctypes
    buf = ctypes.create_string_buffer(64)

    def fd(v):
        assert L.ref_format_double(float(v), buf, 64) == 0
        return buf.value.decode()

    def fi(v):
        assert L.ref_format_int(int(v), buf, 64) == 0
        return buf.value.decode()

    lines = ["id,x,y,z,volume,S_oxygen,U_oxygen,target_oxygen,S_factor,U_factor,target_factor"]
    for k in range(ids.size):
        f = [fi(ids[k])] + [fd(v) for v in pos[k]] + [fd(vol[k])]
        for s in range(2):
            f += [fd(sec[k, s]), fd(upt[k, s]), fd(sat[k, s])]
        lines.append(",".join(f))
    assert p.read_bytes() == ("\n".join(lines) + "\n").encode()


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_parse_matches_reference_on_awkward_tokens(tmp_path):
    w = W.make("t", (10, 10, 10), 2, 0, 1)
    h = "id,x,y,z,volume,S_oxygen,U_oxygen,target_oxygen,S_factor,U_factor,target_factor"
    rows = [
        " 7 ,  0.5, -1e1 ,3.0e+1,2494, 1,0.5e-3,38 ,0,0,0",
        "",                                   # blank lines are skipped
        "-3,.25,5.,-0,1E3,  0 ,10,1,0.000001,2,1",
        "   ",
        "12,99.99999999999999,-100,100,1e-300,5e-324,0,0,1,1,1\r",  # CRLF, subnormal, faces
    ]
    p = tmp_path / "a.csv"
    p.write_text(h + "\n" + "\n".join(rows) + "\n")
    ref = _ref(w)
    want = ref.load_agents(p, NAMES)
    got = B.parse_agents_csv(_mesh(w), p, NAMES)
    for x, y in zip(got, want):
        assert np.array_equal(np.asarray(x).view(np.int64), np.asarray(y).view(np.int64))
    ref.close()


BAD_FILES = {
    "empty": "",
    "header": "id,x,y,z,vol,S_oxygen,U_oxygen,target_oxygen,S_factor,U_factor,target_factor\n",
    "fields": None,
    "number": "1,0,0,0,1x,0,0,0,0,0,0",
    "plus": "1,+1,0,0,1,0,0,0,0,0,0",
    "dup": "1,0,0,0,1,0,0,0,0,0,0\n1,1,1,1,1,0,0,0,0,0,0",
    "volume": "1,0,0,0,0,0,0,0,0,0,0",
    "negative": "1,0,0,0,1,0,-1,0,0,0,0",
    "outside": "1,0,0,1000,1,0,0,0,0,0,0",
    "id": "1.5,0,0,0,1,0,0,0,0,0,0",
}


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", sorted(BAD_FILES) + ["missing"])
def test_errors_match_reference(case, tmp_path):
    w = W.make("t", (10, 10, 10), 2, 0, 1)
    h = "id,x,y,z,volume,S_oxygen,U_oxygen,target_oxygen,S_factor,U_factor,target_factor\n"
    p = tmp_path / f"{case}.csv"
    if case != "missing":
        body = BAD_FILES[case]
        if case == "fields":
            body = "1,0,0,0,1,0,0,0,0,0"
        text = body if case in ("empty", "header") else h + body + "\n"
        p.write_text(text)
    ref = _ref(w)
    with pytest.raises(RefError) as er:
        ref.load_agents(p, NAMES)
    with pytest.raises(B.BiodiffError) as eg:
        B.parse_agents_csv(_mesh(w), p, NAMES)
    assert er.value.code == 1 and isinstance(eg.value, B.ConfigError)  # config_error -> exit code 1
    assert str(eg.value) == str(er.value)[len("[1] "):]
    ref.close()
