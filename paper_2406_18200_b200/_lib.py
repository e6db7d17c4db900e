"""ctypes binding of libseed.so (include/seed.h, include/seed_ops.h): argument marshalling only.

Every computation of the round runs in the CUDA kernels behind these calls; there is no
Python or CPU implementation here, and loading fails loudly when the library is missing.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEED_LIB") or os.path.join(_HERE, "libseed.so")   # SEED_LIB: A/B builds

SEED_OK = 0
STATUS = {0: "SEED_OK", 1: "SEED_EINVAL", 2: "SEED_ENOMEM", 3: "SEED_ECUDA", 4: "SEED_ENCCL",
          5: "SEED_ESTATE", 6: "SEED_ECAPACITY", 7: "SEED_EDEVICE", 8: "SEED_ENOTFOUND"}
FLAG_PROFILE = 1


class SeedError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class ModelShape(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_ff", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


class ModelWeights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("layers", C.POINTER(C.c_void_p)), ("final_norm", C.c_void_p),
                ("lm_head", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("draft", ModelShape), ("target", ModelShape), ("draft_w", ModelWeights), ("target_w", ModelWeights),
                ("gamma", C.c_int32), ("temperature", C.c_float), ("seed", C.c_uint64), ("bonus", C.c_int32),
                ("max_new_tokens", C.c_int32), ("max_streams", C.c_int32), ("max_batch", C.c_int32),
                ("max_ctx", C.c_int32), ("page_tokens", C.c_int32), ("kv_pool_bytes", C.c_int64),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p), ("flags", C.c_uint32),
                ("n_tree", C.c_int32), ("tree_counts", C.c_int32 * 8)]


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_SIGS = {
    # seed.h
    "seed_init": [C.POINTER(Config), C.POINTER(C.c_void_p)],
    "seed_add_stream": [_P, C.c_uint32, _I32P, C.c_int32, _P],
    "seed_schedule_round": [_P, _I32P, C.c_int32, _I32P],
    "seed_draft_round": [_P, _I32P, C.c_int32, _P],
    "seed_verify": [_P, _I32P, C.c_int32, _P, _P, _P],
    "seed_round_host": [_P, _I32P, C.c_int32, _I32P, _I32P, _P],
    "seed_get_tokens": [_P, C.c_uint32, _I32P, C.c_int32, _I32P],
    "seed_stream_info": [_P, C.c_uint32, _I32P],
    "seed_remove_stream": [_P, C.c_uint32],
    "seed_global_pending": [_P, C.POINTER(C.c_int64)],
    "seed_device_status": [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_int64)],
    "seed_fork_stream": [_P, C.c_uint32, C.c_uint32, _P],
    "seed_forward_logits": [_P, C.c_int32, _I32P, C.c_int32, _P, _P],
    "seed_last_round_buffers": [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)],
    "seed_get_profile": [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                         C.POINTER(C.c_int64), C.POINTER(C.c_double)],
    "seed_reset_profile": [_P],
    "seed_set_profile": [_P, C.c_int32],
    "seed_gemm_trace": [_P, C.POINTER(C.c_uint64), C.c_int32, _I32P],
    "seed_gemm_cta_trace": [_P, C.c_int32, C.POINTER(C.c_uint64), _I32P],
    "seed_last_error": [_P],
    "seed_destroy": [_P],
    "seed_nccl_unique_id": [_P],
    "seed_sched_create": [_I32P, C.c_int32, C.POINTER(C.c_void_p)],
    "seed_sched_add": [_P, C.c_int32],
    "seed_sched_pop": [_P, _I32P, C.c_int32, _I32P],
    "seed_sched_complete": [_P, _I32P, _I32P, C.c_int32],
    "seed_sched_all_done": [_P],
    "seed_sched_destroy": [_P],
    "seed_sched_remove": [_P, C.c_int32],
    "seed_table_erase": [_P, C.c_uint32],
    "seed_book_create": [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)],
    "seed_book_add": [_P, C.c_uint32, _I32P, C.c_int32],
    "seed_book_remove": [_P, C.c_uint32],
    "seed_book_schedule": [_P, _I32P, C.c_int32, _I32P],
    "seed_book_pack": [_P, _I32P, C.c_int32, _I32P, _I32P, _I32P],
    "seed_book_complete": [_P, _I32P, C.c_int32],
    "seed_book_global_pending": [_P, C.POINTER(C.c_int64)],
    "seed_book_tokens": [_P, C.c_uint32, _I32P, C.c_int32, _I32P],
    "seed_book_info": [_P, C.c_uint32, _I32P],
    "seed_book_block_ints": [_P],
    "seed_book_destroy": [_P],
    "seed_table_create": [C.c_int32, C.POINTER(C.c_void_p)],
    "seed_table_merge": [_P, _I32P, C.c_int32],
    "seed_table_get": [_P, C.c_uint32, _I32P, C.c_int32, _I32P],
    "seed_table_destroy": [_P],
    # seed_ops.h
    "seed_op_philox": [C.c_uint32] * 6 + [C.c_int32, _P, _P],
    "seed_op_gemm": [_P, C.c_int32, C.c_int32, _P, C.c_int32, _P, _P],
    "seed_op_verify": [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_uint64, _P, _P, C.c_int32,
                       _P, _P, _P, _P, _P, _P],
    "seed_op_draft_sample": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_uint64, _P, _P, C.c_int32, _P,
                             _P],
    "seed_op_draft_topk": [_P, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_uint64, _P, _P, C.c_int32, C.c_int32,
                           _P, C.c_int32, C.c_int32, _P],
    "seed_op_verify_tree": [_P, _P, _P, C.c_int32, _I32P, C.c_int32, C.c_int32, C.c_float, C.c_uint64, _P, _P,
                            C.c_int32, _P, _P, _P, _P],
    "seed_op_decoder_layer": [C.POINTER(ModelShape), C.POINTER(C.c_void_p), _P, C.c_int32, C.c_int32, _P, _P, _P,
                              _P, _P, _P],
    "seed_op_decoder_layer_tree": [C.POINTER(ModelShape), C.POINTER(C.c_void_p), _P, C.c_int32, C.c_int32, _I32P, _P,
                                   _P, _P, _P, _P, _P],
}
_RESTYPE = {"seed_last_error": C.c_char_p, "seed_destroy": None, "seed_sched_destroy": None,
            "seed_table_destroy": None, "seed_sched_all_done": C.c_int32, "seed_book_destroy": None,
            "seed_book_block_ints": C.c_int32}

_lib = None


def load():
    """Load libseed.so (build it first: `python -m paper_2406_18200_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libseed.so not built at {LIB_PATH}; run __graft_entry__.build() -- there is no fallback")
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def check(status, ctx=None, what=""):
    if status != SEED_OK:
        msg = what
        if ctx:
            err = load().seed_last_error(ctx)
            msg = f"{what}: {err.decode() if err else ''}"
        raise SeedError(status, msg)
