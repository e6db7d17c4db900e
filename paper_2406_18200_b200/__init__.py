"""SeeD (arXiv 2406.18200) draft-then-verify round on B200: thin Python binding of libseed.

    from paper_2406_18200_b200 import SeedEngine, ops

SeedEngine wraps seed.h (the round: seed_schedule_round / seed_draft_round / seed_verify);
`ops` wraps seed_ops.h (single kernels, for parity tests).  Torch is used only to own device
memory and to name the current CUDA stream; every step of the path runs in libseed's kernels.
"""
import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import FLAG_PROFILE, SeedError, check

LAYER_KEYS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "attn_norm", "mlp_norm")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _i32(arr):
    a = np.ascontiguousarray(arr, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def model_shape(shape):
    return _lib.ModelShape(vocab=shape["vocab"], d_model=shape["d_model"], n_layers=shape["n_layers"],
                           n_heads=shape["n_heads"], n_kv_heads=shape.get("n_kv_heads", 0), d_ff=shape["d_ff"],
                           rms_eps=shape.get("rms_eps", 1e-5), rope_theta=shape.get("rope_theta", 10000.0))


def _layer_ptrs(L):
    for k in LAYER_KEYS:
        t = L[k]
        if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
            raise ValueError(f"weight {k} must be a contiguous bf16 CUDA tensor")
    return [L[k].data_ptr() for k in LAYER_KEYS]


def _weights(W, keep):
    ptrs = []
    for L in W["layers"]:
        ptrs += _layer_ptrs(L)
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    keep.append(arr)
    return _lib.ModelWeights(embed=W["embed"].data_ptr(), layers=C.cast(arr, C.POINTER(C.c_void_p)),
                             final_norm=W["final_norm"].data_ptr(), lm_head=W["lm_head"].data_ptr())


class SeedEngine:
    """One replica of the round (seed_init ... seed_destroy)."""

    def __init__(self, draft_shape, draft_w, target_shape, target_w, gamma, temperature, seed, bonus=True,
                 max_new=64, max_streams=8, max_batch=8, max_ctx=2048, page_tokens=16, kv_pool_bytes=0,
                 rank=0, world=1, nccl_id=None, profile=False, tree=None):
        self.lib = _lib.load()
        if tree:   # k_config tree rounds (R36): gamma is the tree depth
            gamma = len(tree)
        self.tree = tuple(int(c) for c in tree) if tree else None
        self.gamma, self.vocab = int(gamma), int(target_shape["vocab"])
        keep = []
        cfg = _lib.Config()
        cfg.draft, cfg.target = model_shape(draft_shape), model_shape(target_shape)
        cfg.draft_w, cfg.target_w = _weights(draft_w, keep), _weights(target_w, keep)
        cfg.gamma, cfg.temperature, cfg.seed, cfg.bonus = int(gamma), float(temperature), int(seed), int(bool(bonus))
        cfg.max_new_tokens, cfg.max_streams, cfg.max_batch = int(max_new), int(max_streams), int(max_batch)
        cfg.max_ctx, cfg.page_tokens, cfg.kv_pool_bytes = int(max_ctx), int(page_tokens), int(kv_pool_bytes)
        cfg.rank, cfg.world = int(rank), int(world)
        self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        cfg.nccl_id = C.cast(self._nccl_id, C.c_void_p) if self._nccl_id is not None else None
        cfg.flags = FLAG_PROFILE if profile else 0
        if self.tree:
            cfg.n_tree = len(self.tree)
            for i, c in enumerate(self.tree):
                cfg.tree_counts[i] = c
        torch.cuda.synchronize()
        ctx = C.c_void_p()
        st = self.lib.seed_init(C.byref(cfg), C.byref(ctx))
        if st != 0:
            raise SeedError(st, "seed_init")
        self.ctx = ctx
        self.max_batch = int(max_batch)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.seed_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def _check(self, st, what):
        check(st, self.ctx, what)

    def add_stream(self, gid, prompt, stream=None):
        a, p = _i32(prompt)
        self._check(self.lib.seed_add_stream(self.ctx, int(gid), p, len(a), _stream(stream)), "seed_add_stream")

    def fork_stream(self, src_gid, gid, stream=None):
        self._check(self.lib.seed_fork_stream(self.ctx, int(src_gid), int(gid), _stream(stream)), "seed_fork_stream")

    def schedule(self, cap=None):
        cap = self.max_batch if cap is None else int(cap)
        buf = np.zeros(max(cap, 1), dtype=np.int32)
        n = C.c_int32(0)
        self._check(self.lib.seed_schedule_round(self.ctx, buf.ctypes.data_as(_lib._I32P), cap, C.byref(n)),
                    "seed_schedule_round")
        return buf[:n.value].tolist()

    def draft(self, ids, stream=None):
        a, p = _i32(ids)
        self._check(self.lib.seed_draft_round(self.ctx, p, len(a), _stream(stream)), "seed_draft_round")

    def verify(self, ids, out_tok=None, out_cnt=None, stream=None):
        a, p = _i32(ids)
        self._check(self.lib.seed_verify(self.ctx, p, len(a), _ptr(out_tok), _ptr(out_cnt), _stream(stream)),
                    "seed_verify")

    def round_host(self, ids, stream=None):
        a, p = _i32(ids)
        tok = np.zeros((len(a), self.gamma + 1), dtype=np.int32)
        cnt = np.zeros(len(a), dtype=np.int32)
        self._check(self.lib.seed_round_host(self.ctx, p, len(a), tok.ctypes.data_as(_lib._I32P),
                                             cnt.ctypes.data_as(_lib._I32P), _stream(stream)), "seed_round_host")
        return tok, cnt

    def tokens(self, gid, cap=1 << 16):
        buf = np.zeros(cap, dtype=np.int32)
        n = C.c_int32(0)
        self._check(self.lib.seed_get_tokens(self.ctx, int(gid), buf.ctypes.data_as(_lib._I32P), cap, C.byref(n)),
                    "seed_get_tokens")
        return buf[:n.value].tolist()

    def stream_info(self, gid):
        info = np.zeros(8, dtype=np.int32)
        self._check(self.lib.seed_stream_info(self.ctx, int(gid), info.ctypes.data_as(_lib._I32P)), "seed_stream_info")
        keys = ("T_len", "L", "r", "done", "len_t", "len_d", "pages", "slot")
        return dict(zip(keys, info.tolist()))

    def remove_stream(self, gid):
        self._check(self.lib.seed_remove_stream(self.ctx, int(gid)), "seed_remove_stream")

    def global_pending(self):
        """Streams undone on all ranks after the last completed round (seed_global_pending)."""
        n = C.c_int64(0)
        self._check(self.lib.seed_global_pending(self.ctx, C.byref(n)), "seed_global_pending")
        return n.value

    def device_status(self):
        """(error bits seen since init, K4 empty-residual fallbacks) -- seed_device_status."""
        bits, fb = C.c_uint32(0), C.c_int64(0)
        self._check(self.lib.seed_device_status(self.ctx, C.byref(bits), C.byref(fb)), "seed_device_status")
        return bits.value, fb.value

    def forward_logits(self, which, tokens, stream=None):
        a, p = _i32(tokens)
        out = torch.empty((len(a), self.vocab), dtype=torch.float32, device="cuda")
        self._check(self.lib.seed_forward_logits(self.ctx, int(which), p, len(a), _ptr(out), _stream(stream)),
                    "seed_forward_logits")
        return out

    def last_round(self, n):
        """(target logits [n][g+1][V], draft logits [n][g][V], draft tokens [n][g]) copies (device);
        tree rounds: (target [n][rows][V], draft [n][rows][V], root + node tokens [n][rows])."""
        t, d, x = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(self.lib.seed_last_round_buffers(self.ctx, C.byref(t), C.byref(d), C.byref(x)), "buffers")
        g, V = self.gamma, self.vocab
        if self.tree:
            rows, lvl = 1, 1
            for c in self.tree:
                lvl *= c
                rows += lvl
            return (_wrap(t.value, (n, rows, V), torch.float32), _wrap(d.value, (n, rows, V), torch.float32),
                    _wrap(x.value, (n, rows), torch.int32))
        return (_wrap(t.value, (n, g + 1, V), torch.float32), _wrap(d.value, (n, g, V), torch.float32),
                _wrap(x.value, (n, g), torch.int32))

    def profile(self):
        ms, n, by, k, sp = C.c_double(), C.c_int64(), C.c_double(), C.c_int64(), C.c_double()
        self._check(self.lib.seed_get_profile(self.ctx, C.byref(ms), C.byref(n), C.byref(by), C.byref(k), C.byref(sp)),
                    "profile")
        return {"gemm_ms": ms.value, "gemm_launches": n.value, "gemm_bytes": by.value, "kernel_launches": k.value,
                "gemm_span_ms": sp.value}

    def gemm_trace(self, cap=4096):
        """[(start, release, end)] globaltimer ns of each GEMM launch of the last round (profile=True)."""
        buf = np.zeros(4 * cap, dtype=np.uint64)
        n = C.c_int32(0)
        self._check(self.lib.seed_gemm_trace(self.ctx, buf.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n)),
                    "seed_gemm_trace")
        return buf[:4 * n.value].reshape(-1, 4)[:, :3].astype(np.int64)

    def launch_trace(self, cap=8192):
        """[(start, release, end, kind)] globaltimer ns of every traced launch of the last round
        (profile=True): kind 1 = K2 GEMM, 2 = K3 attention; rows in launch order."""
        buf = np.zeros(4 * cap, dtype=np.uint64)
        n = C.c_int32(0)
        self._check(self.lib.seed_gemm_trace(self.ctx, buf.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n)),
                    "seed_gemm_trace")
        return buf[:4 * n.value].reshape(-1, 4).astype(np.int64)

    def gemm_cta_trace(self, launch):
        """Raw per-CTA phase words (8192) of one launch (profile=True, SEED_CTA_TRACE=1); see seed.h."""
        buf = np.zeros(8192, dtype=np.uint64)
        n = C.c_int32(0)
        self._check(self.lib.seed_gemm_cta_trace(self.ctx, int(launch), buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                 C.byref(n)), "seed_gemm_cta_trace")
        return buf[:n.value].astype(np.int64)

    def set_profile(self, on):
        """Timing records on / off between rounds (the engine must be created with profile=True)."""
        self._check(self.lib.seed_set_profile(self.ctx, int(bool(on))), "seed_set_profile")

    def reset_profile(self):
        self._check(self.lib.seed_reset_profile(self.ctx), "reset_profile")


class _DevView:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    _TYPESTR = {torch.float32: "<f4", torch.int32: "<i4"}

    def __init__(self, ptr, shape, dtype):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": self._TYPESTR[dtype],
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _wrap(ptr, shape, dtype):
    """Copy a library-owned device buffer into a fresh torch tensor."""
    return torch.as_tensor(_DevView(ptr, shape, dtype), device="cuda").clone()


def nccl_unique_id():
    buf = C.create_string_buffer(128)
    check(_lib.load().seed_nccl_unique_id(buf), None, "seed_nccl_unique_id")
    return buf.raw


class Scheduler:
    """Host FCFS rounds scheduler of libseed (seed_sched_*), usable without a GPU."""

    def __init__(self, ids):
        self.lib = _lib.load()
        a, p = _i32(sorted(ids) if ids else [])
        h = C.c_void_p()
        check(self.lib.seed_sched_create(p, len(a), C.byref(h)), None, "seed_sched_create")
        self.h = h

    def add(self, gid):
        check(self.lib.seed_sched_add(self.h, int(gid)), None, "seed_sched_add")

    def pop(self, cap):
        buf = np.zeros(max(cap, 1), dtype=np.int32)
        n = C.c_int32(0)
        st = self.lib.seed_sched_pop(self.h, buf.ctypes.data_as(_lib._I32P), int(cap), C.byref(n))
        check(st, None, "seed_sched_pop")
        return buf[:n.value].tolist()

    def complete(self, batch, done):
        a, p = _i32(batch)
        d, q = _i32([int(bool(x)) for x in done])
        check(self.lib.seed_sched_complete(self.h, p, q, len(a)), None, "seed_sched_complete")

    def all_done(self):
        return bool(self.lib.seed_sched_all_done(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.seed_sched_destroy(self.h)
            self.h = None


class TokenTable:
    """a6 record merge (seed_table_*), usable without a GPU."""

    def __init__(self, gamma):
        self.lib = _lib.load()
        self.stride = gamma + 3
        h = C.c_void_p()
        check(self.lib.seed_table_create(self.stride, C.byref(h)), None, "seed_table_create")
        self.h = h

    def merge(self, records):
        a, p = _i32(np.asarray(records).reshape(-1))
        check(self.lib.seed_table_merge(self.h, p, len(a) // self.stride), None, "seed_table_merge")

    def get(self, gid, cap=1 << 16):
        buf = np.zeros(cap, dtype=np.int32)
        n = C.c_int32(0)
        check(self.lib.seed_table_get(self.h, int(gid), buf.ctypes.data_as(_lib._I32P), cap, C.byref(n)), None,
              "seed_table_get")
        return buf[:n.value].tolist()

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.seed_table_destroy(self.h)
            self.h = None


class RoundBook:
    """One rank's host round bookkeeping (seed_book_*): scheduler, own streams' tokens, the exchange
    block of the per-round all-gather and its merge.  Usable without a GPU (multi-rank CPU tests)."""

    def __init__(self, gamma, max_new, cap, world=1, rank=0):
        self.lib = _lib.load()
        self.gamma = int(gamma)
        h = C.c_void_p()
        check(self.lib.seed_book_create(int(gamma), int(max_new), int(cap), int(world), int(rank), C.byref(h)), None,
              "seed_book_create")
        self.h = h
        self.block_ints = int(self.lib.seed_book_block_ints(h))

    def add(self, gid, prefix):
        a, p = _i32(prefix)
        check(self.lib.seed_book_add(self.h, int(gid), p, len(a)), None, "seed_book_add")

    def remove(self, gid):
        check(self.lib.seed_book_remove(self.h, int(gid)), None, "seed_book_remove")

    def schedule(self, cap):
        buf = np.zeros(max(int(cap), 1), dtype=np.int32)
        n = C.c_int32(0)
        check(self.lib.seed_book_schedule(self.h, buf.ctypes.data_as(_lib._I32P), int(cap), C.byref(n)), None,
              "seed_book_schedule")
        return buf[:n.value].tolist()

    def pack(self, ids, out_tok, out_cnt):
        a, p = _i32(ids)
        t, tp = _i32(np.asarray(out_tok, dtype=np.int32).reshape(-1) if len(a) else np.zeros(1, np.int32))
        c, cp = _i32(out_cnt if len(a) else [0])
        blk = np.zeros(self.block_ints, dtype=np.int32)
        check(self.lib.seed_book_pack(self.h, p, len(a), tp, cp, blk.ctypes.data_as(_lib._I32P)), None,
              "seed_book_pack")
        return blk

    def complete(self, blocks):
        b = np.ascontiguousarray(blocks, dtype=np.int32).reshape(-1)
        check(self.lib.seed_book_complete(self.h, b.ctypes.data_as(_lib._I32P), b.size // self.block_ints), None,
              "seed_book_complete")

    def global_pending(self):
        n = C.c_int64(0)
        check(self.lib.seed_book_global_pending(self.h, C.byref(n)), None, "seed_book_global_pending")
        return n.value

    def tokens(self, gid, cap=1 << 16):
        buf = np.zeros(cap, dtype=np.int32)
        n = C.c_int32(0)
        check(self.lib.seed_book_tokens(self.h, int(gid), buf.ctypes.data_as(_lib._I32P), cap, C.byref(n)), None,
              "seed_book_tokens")
        return buf[:n.value].tolist()

    def info(self, gid):
        info = np.zeros(5, dtype=np.int32)
        check(self.lib.seed_book_info(self.h, int(gid), info.ctypes.data_as(_lib._I32P)), None, "seed_book_info")
        return dict(zip(("T_len", "L", "r", "done", "prompt_len"), info.tolist()))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.seed_book_destroy(self.h)
            self.h = None


from . import ops  # noqa: E402

__all__ = ["SeedEngine", "Scheduler", "TokenTable", "RoundBook", "ops", "SeedError", "nccl_unique_id", "LAYER_KEYS"]
