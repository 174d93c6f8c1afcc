"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, rejects bad arguments synchronously and answers workspace
queries (SURVEY §8(b) conventions)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "symnmf.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2402_08134_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        from paper_2402_08134_b200.build import build
        build()
    return _abi.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(symnmf_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ("symnmf_gram", "symnmf_ah", "symnmf_leverage_scores", "symnmf_hybrid_sample", "symnmf_sampled_ah",
              "symnmf_rangefinder", "symnmf_hals_sweep", "symnmf_iterate"):
        assert n in names


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2402_08134_b200 import _abi
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _abi.SIGNATURES, name


def test_no_product_import_of_oracle():
    pkg = os.path.join(ROOT, "paper_2402_08134_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f


def test_version_and_arg_validation(lib):
    assert lib.symnmf_version() >= 100
    sz = C.c_size_t(0)
    F, G = C.c_void_p(256), C.c_void_p(512)
    assert lib.symnmf_gram(None, 10, 4, G, None, C.byref(sz), None) == 1        # null F
    assert lib.symnmf_gram(F, 0, 4, G, None, C.byref(sz), None) == 1           # n < 1
    assert lib.symnmf_gram(F, 10, 65, G, None, C.byref(sz), None) == 1         # k > 64
    assert lib.symnmf_gram(F, 10, 4, G, None, None, None) == 1                 # no ws_bytes
    assert lib.symnmf_hals_sweep(G, F, F, F, 10, 4, -1.0, None, None, C.byref(sz), None) == 1   # alpha < 0
    lev = C.c_void_p(1024)
    from paper_2402_08134_b200._abi import Plan
    p = Plan(10, 256, 256, 256, 256, 256, 256)
    assert lib.symnmf_hybrid_sample(lev, 10, 4, 5, 0.0, 0, 0, 0, C.byref(p), None, C.byref(sz), None) == 1  # tau
    assert lib.symnmf_hybrid_sample(lev, 10, 4, 0, 0.5, 0, 0, 0, C.byref(p), None, C.byref(sz), None) == 1  # s
    assert lib.symnmf_hybrid_sample(lev, 10, 4, 5, 0.5, 0, 0, 2, C.byref(p), None, C.byref(sz), None) == 1  # side


def test_csr_3xtf32_mismatch_and_rangefinder_bounds(lib):
    from paper_2402_08134_b200._abi import Matrix
    sz = C.c_size_t(0)
    csr = Matrix(1, 0, 100, 256, 0, 256, 256, 500)
    F, Y = C.c_void_p(256), C.c_void_p(256)
    assert lib.symnmf_ah(C.byref(csr), F, 8, Y, 1, None, C.byref(sz), None) == 1   # 3XTF32 on CSR
    assert lib.symnmf_ah(C.byref(csr), F, 8, Y, 0, None, C.byref(sz), None) == 0   # query ok
    dense = Matrix(0, 0, 100, 256, 100, None, None, 0)
    U, lam = C.c_void_p(256), C.c_void_p(256)
    assert lib.symnmf_rangefinder(C.byref(dense), 97, 2, 0, 0, U, lam, None, C.byref(sz), None) == 1  # l > 96
    assert lib.symnmf_rangefinder(C.byref(dense), 101, 2, 0, 0, U, lam, None, C.byref(sz), None) == 1  # l > n
    assert lib.symnmf_rangefinder(C.byref(csr), 10, 2, 0, 0, U, lam, None, C.byref(sz), None) == 1    # CSR
    assert lib.symnmf_rangefinder(C.byref(dense), 10, 2, 0, 0, U, lam, None, C.byref(sz), None) == 0
    assert sz.value >= 4 * 100 * 10 * 4


def test_workspace_queries_scale_with_n(lib):
    F, G = C.c_void_p(256), C.c_void_p(256)
    s1, s2 = C.c_size_t(0), C.c_size_t(0)
    assert lib.symnmf_leverage_scores(F, 1000, 8, G, None, None, C.byref(s1), None) == 0
    assert lib.symnmf_leverage_scores(F, 10 ** 7, 8, G, None, None, C.byref(s2), None) == 0
    assert s2.value >= s1.value > 0
    from paper_2402_08134_b200._abi import Plan
    p = Plan(10, 256, 256, 256, 256, 256, 256)
    s3 = C.c_size_t(0)
    assert lib.symnmf_hybrid_sample(F, 2_000_000, 32, 20000, 1 / 20000, 0, 0, 0, C.byref(p), None,
                                    C.byref(s3), None) == 0
    assert s3.value >= 2_000_000 * 12                                  # prefix (u64) + multiplicities (i32)


def test_workspace_too_small_is_rejected(lib):
    F, G = C.c_void_p(256), C.c_void_p(256)
    sz = C.c_size_t(0)
    assert lib.symnmf_gram(F, 1000, 8, G, None, C.byref(sz), None) == 0
    small = C.c_size_t(sz.value - 1)
    assert lib.symnmf_gram(F, 1000, 8, G, C.c_void_p(256), C.byref(small), None) == 3   # ERR_WORKSPACE


def test_solver_create_query_without_gpu(lib):
    from paper_2402_08134_b200._abi import Matrix
    dense = Matrix(0, 0, 1000, 256, 1000, None, None, 0)
    W = H = C.c_void_p(256)
    sz = C.c_size_t(0)
    rc = lib.symnmf_solver_create(None, C.byref(dense), 1000, W, H, 8, 1.0, 1, 0, 200, 1 / 200, 0, 0, 20,
                                  None, None, 0, 0, None, C.byref(sz), None)
    assert rc == 0 and sz.value > 1000 * 8 * 4
    rc = lib.symnmf_solver_create(None, C.byref(dense), 1000, W, H, 8, 1.0, 2, 0, 0, 1.0, 0, 0, 20,
                                  None, None, 0, 0, None, C.byref(sz), None)
    assert rc == 1                                                      # LAI without U / lambda


def test_next_items_argument_validation_without_gpu(lib):
    """NEXT-1/2/3 entry points reject bad arguments synchronously and answer workspace queries."""
    from paper_2402_08134_b200._abi import Matrix, RULE_BPP
    sz = C.c_size_t(0)
    G, Y, F, X = (C.c_void_p(256),) * 4
    # BPP: alpha < 0, k > 64 rejected, query ok
    assert lib.symnmf_bpp_update(G, Y, F, X, 100, 8, -1.0, None, None, None, C.byref(sz), None) == 1
    assert lib.symnmf_bpp_update(G, Y, F, X, 100, 40, 1.0, None, None, None, C.byref(sz), None) == 0   # k <= 64
    assert lib.symnmf_bpp_update(G, Y, F, X, 100, 65, 1.0, None, None, None, C.byref(sz), None) == 1   # k > 64
    assert lib.symnmf_bpp_update(G, Y, F, X, 100, 16, 1.0, None, None, None, C.byref(sz), None) == 0
    dense = Matrix(0, 0, 1000, 256, 1000, None, None, 0)
    csr = Matrix(1, 0, 1000, 256, 0, 256, 256, 5000)
    U, lam = C.c_void_p(256), C.c_void_p(256)
    passes = C.c_int32(0)
    # Ada-RRF: q_max < 1, tol < 0, CSR input
    assert lib.symnmf_rangefinder_adaptive(C.byref(dense), 10, 0, 1e-3, 0, 0, U, lam, C.byref(passes), None, None,
                                           C.byref(sz), None) == 1
    assert lib.symnmf_rangefinder_adaptive(C.byref(dense), 10, 4, -1.0, 0, 0, U, lam, C.byref(passes), None, None,
                                           C.byref(sz), None) == 1
    assert lib.symnmf_rangefinder_adaptive(C.byref(csr), 10, 4, 1e-3, 0, 0, U, lam, C.byref(passes), None, None,
                                           C.byref(sz), None) == 1
    assert lib.symnmf_rangefinder_adaptive(C.byref(dense), 10, 4, 1e-3, 0, 1, U, lam, C.byref(passes), None, None,
                                           C.byref(sz), None) == 0 and sz.value > 4 * 1000 * 10
    # projected gradient: CSR with 3XTF32, bad precision, query ok
    out = C.c_void_p(256)
    assert lib.symnmf_projected_gradient(C.byref(csr), F, 8, 1, out, None, C.byref(sz), None) == 1
    assert lib.symnmf_projected_gradient(C.byref(dense), F, 8, 7, out, None, C.byref(sz), None) == 1
    assert lib.symnmf_projected_gradient(C.byref(dense), F, 8, 0, out, None, C.byref(sz), None) == 0
    # solve: patience < 1, tol < 0; the BPP rule bit is accepted by the solver query
    its = (C.c_int32 * 2)()
    W = H = C.c_void_p(256)
    assert lib.symnmf_solve(C.byref(dense), 1000, W, H, 8, 1.0, 0, 0, 0, 1.0, 0, None, None, 0, 50, 1e-4, 0, 0,
                            its, None, None, C.byref(sz), None) == 1
    assert lib.symnmf_solve(C.byref(dense), 1000, W, H, 8, 1.0, 0, 0, 0, 1.0, 0, None, None, 0, 50, -1.0, 4, 0,
                            its, None, None, C.byref(sz), None) == 1
    assert lib.symnmf_solve(C.byref(dense), 1000, W, H, 8, 1.0, 0 | RULE_BPP, 0, 0, 1.0, 0, None, None, 0, 50, 1e-4,
                            4, 1, its, None, None, C.byref(sz), None) == 0
    assert lib.symnmf_solver_create(None, C.byref(dense), 1000, W, H, 40, 1.0, RULE_BPP, 0, 0, 1.0, 0, 0, 5,
                                    None, None, 0, 0, None, C.byref(sz), None) == 0     # BPP: k <= 64
