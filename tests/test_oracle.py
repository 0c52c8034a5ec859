"""Pins the CPU oracle (oracle/) against the reference's own outputs.

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py); the KATs are the reference's own
(test_rng.py:12-25).  sfc64 is pinned against numpy's SFC64 and its KAT
files; xoshiro256++ against the published algorithm's first outputs for the
state {1, 2, 3, 4} and an independent C restatement (oracle/streams.c).
"""

import ctypes
import os

import numpy as np
import pytest

from conftest import case_config
from oracle import sdeb_oracle as O

# /root/reference/pkg/tests/test_rng.py:12-25
PHILOX_KATS = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ((1, 0, 0, 0), (0, 0), (0xF8E4CCA4, 0x5CB200DB, 0xB1A574EB, 0x097EFF67)),
    ((0, 0, 0, 0), (42, 7), (0x64D43A77, 0xFF08A6BF, 0xFF050829, 0x1E30FA6B)),
    ((123, 456, 789, 1011), (2021, 2022), (0xEE178530, 0xE8ED390A, 0xA30DC0B5, 0x644606D0)),
]

# xoshiro256++ from state {1, 2, 3, 4}: derived by hand from the published
# update (result = rotl(s0 + s3, 23) + s0, ...): 5*2**23 + 1 = 41943041, ...
XOSHIRO_KAT = [41943041, 58720359, 3588806011781223, 3591011842654386]


@pytest.mark.parametrize("counter,key,expected", PHILOX_KATS)
def test_philox_kats(counter, key, expected, cstreams):
    assert O.philox_block(counter, key) == expected
    assert tuple(int(w) for w in O.philox_words(key[0], key[1], *counter)) == expected
    out = (ctypes.c_uint32 * 4)()
    cstreams.oracle_philox((ctypes.c_uint32 * 4)(*counter), (ctypes.c_uint32 * 2)(*key), out)
    assert tuple(out) == expected


def test_philox_words_golden(golden):
    arrays, _ = golden
    kc = arrays["philox_in"]
    words = O.philox_words(kc[:, 0], kc[:, 1], kc[:, 2], kc[:, 3], kc[:, 4], kc[:, 5])
    assert np.array_equal(np.stack(words, axis=-1), arrays["philox_out"])


def test_normals_golden(golden):
    arrays, cases = golden
    for idx in range(7):
        c = cases["normals_%d" % idx]
        got = O.normals_for_orbits(int(c["seed"]), np.array(c["orbits"], np.uint32),
                                   c["chunk"], c["step"], c["m"])
        # same op order; only libm dispatch of the host could differ (<= 1 ulp)
        np.testing.assert_allclose(got, arrays["normals_%d" % idx], rtol=1e-14, atol=1e-15)


def test_normals_prefix_stable():
    full = O.normals_for_orbits(7, np.array([1], np.uint32), 0, 5, 12)
    for m in (1, 4, 5, 11):
        assert np.array_equal(O.normals_for_orbits(7, np.array([1], np.uint32), 0, 5, m),
                              full[:, :m])


def test_sampling_golden(golden):
    arrays, _ = golden
    assert np.array_equal(O.sampling_uniforms(11, np.arange(8), 10), arrays["sampling_uniforms"])
    init, params = O.sample_kuramoto_batch(16, 64, (0.2, 0.4), (0.01, 0.03), 0.25, seed=99)
    assert np.array_equal(init, arrays["sample_init"])
    assert np.array_equal(params, arrays["sample_params"])
    init, params = O.sample_kuramoto_batch(4, 32, (0.01, 0.03), (0.001, 0.003), 1.0,
                                           seed=20260809)
    assert np.array_equal(init, arrays["speed_init"])
    assert np.array_equal(params, arrays["speed_params"])


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16, 33, 64])
def test_drift_golden(golden, n):
    arrays, _ = golden
    got = O.kuramoto_drift(arrays["drift_y_%d" % n], arrays["drift_p_%d" % n])
    np.testing.assert_allclose(got, arrays["drift_f_%d" % n], rtol=1e-14, atol=1e-15)


def test_drift_hand_example():
    # /root/reference/pkg/tests/test_model.py:21-25
    f = O.kuramoto_drift(np.array([0.0, np.pi / 2]), np.array([1.0, 0.1, 0.2, 0.0, 0.0]))
    np.testing.assert_allclose(f, [0.6, -0.3], atol=1e-12)


STORE_CASES = ["cfg1", "engine5", "engine5_k4", "cfg2", "n33", "n64", "n256", "rk4_8",
               "euler_8", "em0_8", "failures", "pad", "rotator", "accept7"]


def run_oracle_case(arrays, case, name, **kw):
    cfg = case_config(case)
    chunks = O.iteration_count(cfg["tspan"], cfg["dt"], cfg["ksteps"], cfg["pad"])
    return O.integrate(arrays[name + "_init"], arrays[name + "_params"], dt=cfg["dt"],
                       ksteps=cfg["ksteps"], chunks=chunks, seed=cfg["seed"],
                       solver=cfg["solver"], nnoise=case["nnoise"], **kw)


@pytest.mark.parametrize("name", STORE_CASES)
def test_restated_loop_matches_run_batch(golden, name):
    arrays, cases = golden
    case = cases[name]
    times, values, failures = run_oracle_case(arrays, case, name)
    assert np.array_equal(times, arrays[name + "_times"])
    # same op order as run_batch: bit-identical on this host; other hosts'
    # libm may move the last ulp, hence the (much tighter than 1e-10) bound
    assert O.mixed_error(values, arrays[name + "_values"]) <= 1e-12
    assert [list(f) for f in failures] == case["failures"]


def test_restated_loop_shard_offsets(golden):
    # rows 32..63 of a 64-orbit run_batch == the oracle on global ids 32..63 alone
    arrays, cases = golden
    case = cases["cfg1"]
    cfg = case_config(case)
    chunks = O.iteration_count(cfg["tspan"], cfg["dt"], cfg["ksteps"])
    _, values, _ = O.integrate(arrays["cfg1_init"][32:], arrays["cfg1_params"][32:],
                               dt=cfg["dt"], ksteps=cfg["ksteps"], chunks=chunks,
                               seed=cfg["seed"], orbit_ids=np.arange(32, 64))
    assert O.mixed_error(values, arrays["cfg1_values"][32:]) <= 1e-12


def test_restated_loop_group_and_thread_invariance(golden):
    arrays, cases = golden
    case = cases["engine5"]
    a = run_oracle_case(arrays, case, "engine5")[1]
    b = run_oracle_case(arrays, case, "engine5", threads=4, group=3)[1]
    assert np.array_equal(a, b)


# ---- sfc64 / xoshiro256++ ----------------------------------------------------

def _numpy_kat(name):
    path = os.path.join(os.path.dirname(np.__file__), "random", "tests", "data", name)
    if not os.path.exists(path):
        pytest.skip("numpy KAT file %s not installed" % name)
    lines = [ln for ln in open(path).read().split("\n") if ln.strip()]
    seed = int(lines[0].split(",")[1], 16 if "0x" in lines[0] else 10)
    return seed, [int(ln.split(",")[1], 16) for ln in lines[1:]]


@pytest.mark.parametrize("kat", ["sfc64-testset-1.csv", "sfc64-testset-2.csv"])
def test_sfc64_numpy_kat(kat, cstreams):
    seed, expected = _numpy_kat(kat)
    seed3 = np.random.SeedSequence(seed).generate_state(3, np.uint64)
    s = O.sfc64_seed_words(seed3[0:1], seed3[1:2], seed3[2:3])
    got = [int(O.sfc64_next(s)[0]) for _ in range(len(expected))]
    assert got == expected
    st = np.zeros(4, np.uint64)
    cstreams.oracle_sfc64_set_seed(np.ascontiguousarray(seed3).ctypes.data_as(
        ctypes.POINTER(ctypes.c_uint64)), st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    out = np.zeros(len(expected), np.uint64)
    cstreams.oracle_stream_raw_from_state(1, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                          len(expected),
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert [int(x) for x in out] == expected


def test_sfc64_matches_numpy_bit_generator():
    # our per-(orbit, block) state, loaded into numpy's SFC64, gives the same outputs
    s = O.stream_init("sfc64", 12345, np.array([7], np.uint64), np.array([3], np.uint64))
    g = np.random.SFC64()
    g.state = {"bit_generator": "SFC64",
               "state": {"state": np.array([int(w[0]) for w in s], dtype=np.uint64)},
               "has_uint32": 0, "uinteger": 0}
    ours = [int(O.sfc64_next(s)[0]) for _ in range(64)]
    assert ours == [int(x) for x in g.random_raw(64)]


def test_xoshiro_kat(cstreams):
    s = [np.array([v], np.uint64) for v in (1, 2, 3, 4)]
    assert [int(O.xoshiro256pp_next(s)[0]) for _ in range(4)] == XOSHIRO_KAT
    st = np.array([1, 2, 3, 4], np.uint64)
    out = np.zeros(4, np.uint64)
    cstreams.oracle_stream_raw_from_state(2, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                          4, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    assert [int(x) for x in out] == XOSHIRO_KAT


@pytest.mark.parametrize("stream,sid", [("sfc64", 1), ("xoshiro256pp", 2)])
def test_stream_restatements_agree(stream, sid, cstreams):
    for seed, orbit, block in [(0, 0, 0), (2 ** 64 - 1, 2 ** 32 - 1, 63), (20260809, 5, 2)]:
        py = O.stream_raw(stream, seed, orbit, block, 100)
        out = np.zeros(100, np.uint64)
        cstreams.oracle_stream_raw(sid, seed, orbit, block, 100,
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        assert np.array_equal(py, out)


def test_stream_normals_moments():
    # per-(orbit, block) streams give standard normals (cf. test_rng.py:162-171)
    for stream in ("sfc64", "xoshiro256pp"):
        st = O.stream_init(stream, 123, np.arange(2500, dtype=np.uint64)[:, None],
                           np.zeros((1, 1), np.uint64))
        draws = np.concatenate([O.gaussian_from_words(*O.stream_block_words(stream, st), 4).ravel()
                                for _ in range(100)])
        assert draws.size == 1_000_000
        assert abs(draws.mean()) < 0.01
        assert abs(draws.var() - 1.0) < 0.01


def test_stream_blocks_are_distinct():
    w = O.stream_block_words("sfc64", O.stream_init("sfc64", 0, np.arange(64, dtype=np.uint64)[:, None],
                                                     np.arange(4, dtype=np.uint64)[None, :]))
    stacked = np.stack([x.ravel() for x in w], axis=-1)
    assert np.unique(stacked, axis=0).shape[0] == 256
