"""Pin of the oracle's multi-way contraction at the full C3 sketch width (w = 4096).

The oracle evaluates multi-way sub-plans by exact message passing with the min-abs
contraction identity (oracle/compass_oracle.c or_contract_row), the same
reformulation the GPU engine uses, and its literal-definition twin (or_contract_brute_row)
only reaches w <= ~5.  Here every one of the 14 connected sub-plans of the C3 join graph
(the paper's running example shape) is evaluated at w = 4096 a second,
independent way: merged views are materialised (left fold in canonical
edge order) and the definition E = sum over bucket assignments of the product of the tables'
tensors is summed densely, factored only by distributivity (tests/dense_pin.c,
numpy for the O(w^2) sums).  No sorting, no thresholds, no prefix sums.

Values are drawn from [-1000, 1000] (heavy ties, zeros) so the dense int64 inner sums are
exact.  CPU only; ~1 min on 8 cores (the w^3 sums run on all cores).
"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
W = 4096
E1, E2, E3, E4, E5 = "K.id|MK.kid", "MK.mid|T.id", "CI.mid|T.id", "CI.mid|MK.mid", "CI.pid|N.id"


@pytest.fixture(scope="module")
def dense():
    out = os.path.join(tempfile.mkdtemp(), "dense_pin.so")
    subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC",
                    os.path.join(HERE, "dense_pin.c"), "-o", out], check=True)
    L = ctypes.CDLL(out)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.dp_merged3_contract.argtypes = [vp, vp, vp, ctypes.c_int, vp, i64, vp]
    L.dp_merged2.argtypes = [vp, vp, i64, vp]
    L.dp_triangle.argtypes = [vp, vp, vp, i64, vp]
    return L


def _p(a):
    return a.ctypes.data


@pytest.fixture(scope="module")
def vecs():
    rng = np.random.default_rng(20210204)
    v = {}
    for key in ["K1", "MK1", "MK2", "MK4", "T2", "T3", "CI3", "CI4", "CI5", "N5"]:
        a = rng.integers(-1000, 1001, W).astype(np.int64)
        a[rng.random(W) < 0.1] = 0
        a[:8] = [5, -5, 5, 0, 1000, -1000, 3, -3]      # exact |.| ties across constituents
        v[key] = a
    return v


def _graph(v):
    vec = {("K", E1): v["K1"], ("MK", E1): v["MK1"], ("MK", E2): v["MK2"], ("MK", E4): v["MK4"],
           ("T", E2): v["T2"], ("T", E3): v["T3"], ("CI", E3): v["CI3"], ("CI", E4): v["CI4"],
           ("CI", E5): v["CI5"], ("N", E5): v["N5"]}
    vec = {k: a.reshape(1, W) for k, a in vec.items()}
    edges = [(E1, "K", "MK"), (E2, "MK", "T"), (E3, "CI", "T"), (E4, "CI", "MK"), (E5, "CI", "N")]
    return oracle.Graph({t: 1 for t in ["K", "MK", "T", "CI", "N"]}, edges, vec)


def _m(L, u, v):
    M = np.empty((W, W), dtype=np.int64)
    L.dp_merged2(_p(u), _p(v), W, _p(M))
    return M


def _m3(L, v0, v1, v2, q, x):
    out = np.empty((W, W), dtype=np.int64)
    L.dp_merged3_contract(_p(v0), _p(v1), _p(v2), q, _p(x), W, _p(out))
    return out


def _tri(L, A, B, C):
    lohi = np.zeros(2, dtype=np.int64)
    L.dp_triangle(_p(np.ascontiguousarray(A)), _p(np.ascontiguousarray(B)), _p(np.ascontiguousarray(C)), W, _p(lohi))
    return int(lohi[0]) % (1 << 64) + int(lohi[1]) * (1 << 64)


def _dot(a, b):
    return sum(int(x) for x in (a.astype(object) * b.astype(object)))


def _vm(x, M):
    """x^T M over int64 (exact: |x| <= 1000, |M| <= 1000, w = 4096)."""
    return x @ M


def dense_truth(L, v):
    """E for every connected sub-plan of C3, canonical order E4 < E3 < E5 < E1 < E2."""
    K1, MK1, MK2, MK4 = v["K1"], v["MK1"], v["MK2"], v["MK4"]
    T2, T3, CI3, CI4, CI5, N5 = v["T2"], v["T3"], v["CI3"], v["CI4"], v["CI5"], v["N5"]
    out = {}
    out[("K", "MK")] = _dot(K1, MK1)
    out[("MK", "T")] = _dot(MK2, T2)
    out[("CI", "MK")] = _dot(MK4, CI4)
    out[("CI", "T")] = _dot(T3, CI3)
    out[("CI", "N")] = _dot(CI5, N5)
    # 3-table chains through a merged 2-constituent view (O(w^2) dense)
    out[("K", "MK", "T")] = _dot(_vm(K1, _m(L, MK1, MK2)), T2)           # <MK_e1, MK_e2>[i][j]
    out[("CI", "K", "MK")] = _dot(_vm(CI4, _m(L, MK4, MK1)), K1)          # <MK_e4, MK_e1>[l][i]
    out[("CI", "MK", "N")] = _dot(_vm(MK4, _m(L, CI4, CI5)), N5)          # <CI_e4, CI_e5>[l][k]
    out[("CI", "N", "T")] = _dot(_vm(T3, _m(L, CI3, CI5)), N5)            # <CI_e3, CI_e5>[j][k]
    # triangle {MK, T, CI}: edges e2 (j2), e3 (j3), e4 (l)
    Tm = _m(L, T3, T2)        # <T_e3, T_e2>[j3][j2]
    MKm = _m(L, MK4, MK2)     # <MK_e4, MK_e2>[l][j2]
    CIm = _m(L, CI4, CI3)     # <CI_e4, CI_e3>[l][j3]
    out[("CI", "MK", "T")] = _tri(L, MKm, Tm, CIm)
    # {K, MK, CI, N}: edges e1, e4, e5
    a = _m(L, MK4, MK1) @ K1                # sum_i <MK_e4, MK_e1>[l][i] K1[i]  -> vector over l
    b = _m(L, CI4, CI5) @ N5                # sum_k <CI_e4, CI_e5>[l][k] N5[k] -> vector over l
    out[("CI", "K", "MK", "N")] = _dot(a, b)
    # 3-constituent views with one leg contracted against a vector leaf (w^3)
    MKp = _m3(L, MK4, MK1, MK2, 1, K1)      # sum_i K1[i] fold(MK_e4[l], MK_e1[i], MK_e2[j2]) -> [l][j2]
    CIp = _m3(L, CI4, CI3, CI5, 2, N5)      # sum_k fold(CI_e4[l], CI_e3[j3], CI_e5[k]) N5[k] -> [l][j3]
    out[("CI", "K", "MK", "T")] = _tri(L, MKp, Tm, CIm)
    out[("CI", "MK", "N", "T")] = _tri(L, MKm, Tm, CIp)
    out[("CI", "K", "MK", "N", "T")] = _tri(L, MKp, Tm, CIp)
    return out


@pytest.mark.slow
def test_c3_all_14_subplans_full_width_dense_definition(dense, vecs):
    g = _graph(vecs)
    truth = dense_truth(dense, vecs)
    assert len(truth) == 14
    subs = oracle.connected_subplans(g)
    assert sorted(tuple(sorted(s)) for s in subs) == sorted(tuple(sorted(k)) for k in truth)
    for s in subs:
        key = tuple(sorted(s))
        rows = oracle.estimate_rows(g, key)
        assert rows == [truth[key]], (key, rows, truth[key])
