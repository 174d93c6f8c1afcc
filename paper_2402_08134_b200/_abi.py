"""ctypes view of include/symnmf.h (argument marshalling only).

Loads the in-tree libsymnmf.so and fails loudly if it is missing: there is no
CPU or PyTorch fallback for any operation of the hot path.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsymnmf.so")

OK, ERR_ARG, ERR_NOT_PD, ERR_WORKSPACE, ERR_CUDA, ERR_UNSUPPORTED, ERR_CAPACITY = range(7)
STATUS_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_NOT_PD", 3: "ERR_WORKSPACE", 4: "ERR_CUDA",
                5: "ERR_UNSUPPORTED", 6: "ERR_CAPACITY"}
DENSE, CSR = 0, 1
FP32, TF32X3 = 0, 1
EXACT, LVS, LAI = 0, 1, 2
RULE_BPP = 16
RECORD_PLANS = 32

# name -> (restype, argtypes); the authoritative list of exported entry points.
P = C.c_void_p
I32, I64, U32, U64, F64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
PSZ = C.POINTER(C.c_size_t)


class Matrix(C.Structure):
    _fields_ = [("kind", I32), ("reserved", I32), ("n", I64), ("val", P), ("lda", I64),
                ("rowptr", P), ("colidx", P), ("nnz", I64)]


class Plan(C.Structure):
    _fields_ = [("cap", I64), ("det_idx", P), ("draw_idx", P), ("uniq_idx", P), ("uniq_w", P),
                ("counts", P), ("mass", P)]


class HalfStats(C.Structure):
    _fields_ = [("s_d", I64), ("s_r", I64), ("n_uniq", I64), ("theta", F64)]


PM = C.POINTER(Matrix)
PP = C.POINTER(Plan)

SIGNATURES = {
    "symnmf_version": (I32, []),
    "symnmf_status_read": (I32, [P, C.POINTER(I32), P]),
    "symnmf_gram": (I32, [P, I64, I32, P, P, PSZ, P]),
    "symnmf_ah": (I32, [PM, P, I32, P, I32, P, PSZ, P]),
    "symnmf_leverage_scores": (I32, [P, I64, I32, P, P, P, PSZ, P]),
    "symnmf_hybrid_sample": (I32, [P, I64, I32, I64, F64, U64, U32, U32, PP, P, PSZ, P]),
    "symnmf_sampled_ah": (I32, [PM, P, I32, PP, P, P, P, PSZ, P]),
    "symnmf_rangefinder": (I32, [PM, I32, I32, U64, I32, P, P, P, PSZ, P]),
    "symnmf_gaussian": (I32, [I64, I32, U64, P, P]),
    "symnmf_rangefinder_adaptive": (I32, [PM, I32, I32, F64, U64, I32, P, P, C.POINTER(I32), C.POINTER(F64), P,
                                          PSZ, P]),
    "symnmf_lai_ah": (I32, [P, P, I64, I32, P, I32, P, P, PSZ, P]),
    "symnmf_hals_sweep": (I32, [P, P, P, P, I64, I32, F64, P, P, PSZ, P]),
    "symnmf_residual": (I32, [PM, P, I32, P, P, PSZ, P]),
    "symnmf_bpp_update": (I32, [P, P, P, P, I64, I32, F64, P, C.POINTER(I32), P, PSZ, P]),
    "symnmf_projected_gradient": (I32, [PM, P, I32, I32, P, P, PSZ, P]),
    "symnmf_iterate": (I32, [PM, I64, P, P, I32, F64, I32, I32, I64, F64, U64, I32, I32, P, P, I32,
                             C.POINTER(HalfStats), C.POINTER(F64), P, PSZ, P]),
    "symnmf_solver_create": (I32, [C.POINTER(P), PM, I64, P, P, I32, F64, I32, I32, I64, F64, U64, I32, I32,
                                   P, P, I32, I32, P, PSZ, P]),
    "symnmf_solver_run": (I32, [P, I32, P]),
    "symnmf_solver_stats": (I32, [P, C.POINTER(I32), C.POINTER(HalfStats), C.POINTER(F64), P]),
    "symnmf_solver_destroy": (I32, [P]),
    "symnmf_solver_run_until": (I32, [P, I32, F64, I32, C.POINTER(I32), P]),
    "symnmf_solver_pgrad": (I32, [P, C.POINTER(F64), P]),
    "symnmf_solve": (I32, [PM, I64, P, P, I32, F64, I32, I32, I64, F64, U64, P, P, I32, I32, F64, I32, I32,
                           C.POINTER(I32), C.POINTER(F64), P, PSZ, P]),
    "symnmf_solver_last_plan": (I32, [P, P, P, P, P, P, P]),
    "symnmf_solver_plan_history": (I32, [P, I32, I32, P, P, P, P, P, P]),
    "symnmf_solver_graph_nodes": (I32, [P, C.POINTER(I32), C.POINTER(I32)]),
    "symnmf_solver_profile": (I32, [P, I32, I32, C.c_void_p, C.POINTER(C.c_float), C.POINTER(I32), P]),
    "symnmf_leverage_scores_gram": (I32, [P, I64, I32, P, P, P, PSZ, P]),
    "symnmf_hybrid_shard_sums": (I32, [P, I64, I32, F64, P, P, P, P, PSZ, P]),
    "symnmf_hybrid_shard_plan": (I32, [P, I64, I64, I32, I64, F64, U64, U32, U32, U64, U64, I64, PP, P, PSZ, P]),
    "symnmf_plan_rows_scaled": (I32, [P, I64, I32, PP, P, P, P, PSZ, P]),
    "symnmf_sampled_ah_rows": (I32, [PM, I64, P, P, I64, P, I32, P, P, PSZ, P]),
    "symnmf_lai_project_rows": (I32, [P, I64, I32, P, I32, P, P, PSZ, P]),
    "symnmf_lai_apply_rows": (I32, [P, P, I64, I32, P, I32, P, P, PSZ, P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libsymnmf.so and bind every declared entry point (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libsymnmf.so not built at {path}: run __graft_entry__.build() "
                          "(python -m paper_2402_08134_b200.build); there is no fallback path")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class SymNMFError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} returned {STATUS_NAMES.get(code, code)}")
        self.code = code


def check(fn: str, code: int):
    if code != OK:
        raise SymNMFError(fn, code)
