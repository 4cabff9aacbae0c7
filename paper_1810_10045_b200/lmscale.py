"""Thin ctypes binding of the lmscale C ABI (include/lmscale.h).

Argument marshalling only: every step of the exchange runs in the CUDA
kernels of ``liblmscale.so``.  torch supplies device memory, streams and the
process group used to distribute the NCCL id; there is no CPU fallback -- if
the library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# LMSCALE_LIB selects another in-tree build (e.g. liblmscale_checked.so, the
# device-bounds-checked build); there is no fallback to anything else
LIB_PATH = os.environ.get("LMSCALE_LIB") or os.path.join(_PKG, "liblmscale.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1810_10045_b200._build` "
        "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

OK, INVALID_ARG, ID_RANGE, CUDA_ERR, NCCL_ERR, OOM, UNSUPPORTED, CONSISTENCY = range(8)
FLAG_NO_COMM = 1
FLAG_TIMING = 2
FLAG_GRAPH = 4
FLAG_CHECK = 8

_P = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class Config(ctypes.Structure):
    _fields_ = [("vocab", _i64), ("max_tokens", _i64), ("dim", _i64), ("world", _i32),
                ("rank", _i32), ("device", _i32), ("flags", ctypes.c_uint32)]


class SparseGradC(ctypes.Structure):
    _fields_ = [("ids", _P), ("counts", _P), ("rows", _P), ("num_unique", _i64)]


class StatsC(ctypes.Structure):
    _fields_ = [("u_local", _i64), ("u_global", _i64),
                ("us_dedup", ctypes.c_double), ("us_gather", ctypes.c_double),
                ("us_merge", ctypes.c_double), ("us_scatter", ctypes.c_double),
                ("us_allreduce", ctypes.c_double), ("us_update", ctypes.c_double),
                ("us_total", ctypes.c_double),
                ("bytes_ids_gathered", _i64), ("bytes_grad_allreduce", _i64),
                ("bytes_scatter", _i64), ("bytes_update", _i64), ("workspace_bytes", _i64),
                ("kernels_last_call", _i32), ("kernels_total_lo", _i32),
                ("fused_s5_s6", _i32), ("nvls_available", _i32)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_S = ctypes.c_int
_get_nccl_id = _sig("lmscale_get_nccl_id", _S, [ctypes.c_char_p])
_init = _sig("lmscale_init", _S, [ctypes.POINTER(Config), ctypes.c_char_p, ctypes.POINTER(_P)])
_destroy = _sig("lmscale_destroy", None, [_P])
_unique = _sig("lmscale_unique", _S, [_P, _P, _i64, _P, _P, _P, _P, _P])
_global_unique = _sig("lmscale_global_unique", _S, [_P, _P, _i64, _P])
_scatter_expand = _sig("lmscale_scatter_expand", _S, [_P, _P, _i64, _P])
_get_sparse_grad = _sig("lmscale_get_sparse_grad", _S, [_P, ctypes.POINTER(SparseGradC), _P])
_get_local_maps = _sig("lmscale_get_local_maps", _S,
                       [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P),
                        ctypes.POINTER(_P), ctypes.POINTER(_i64), _P])
_sync = _sig("lmscale_sync_embedding_grad", _S,
             [_P, _P, _P, _i64, ctypes.POINTER(SparseGradC), _P])
_apply = _sig("lmscale_apply_sparse_update", _S,
              [_P, _P, ctypes.POINTER(SparseGradC), ctypes.c_float, _P])
_step = _sig("lmscale_step", _S, [_P, _P, _P, _i64, _P, ctypes.c_float, ctypes.POINTER(_i64), _P])
_emulate_step = _sig("lmscale_emulate_step", _S, [ctypes.POINTER(_P), ctypes.c_int,
                                                  ctypes.POINTER(_P), ctypes.POINTER(_P), _i64,
                                                  ctypes.POINTER(_P), ctypes.c_float, _P])
_dense = _sig("lmscale_sync_dense_baseline", _S, [_P, _P, _P, _i64, _P, ctypes.c_float, _P])
_dense_apply = _sig("lmscale_dense_apply", _S, [_P, _P, _P, _i64, _P, ctypes.c_float, _P])
_host_step = _sig("lmscale_train_step_host", _S,
                  [_P, _P, _P, _i64, _P, ctypes.c_float, _P, ctypes.POINTER(_i64), _P])
_alloc_table = _sig("lmscale_alloc_table", _S, [_P, ctypes.POINTER(_P), ctypes.POINTER(_i64)])
_set_timing = _sig("lmscale_set_timing", _S, [_P, ctypes.c_int])
_plan_seeds = _sig("lmscale_plan_seeds", _S, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                                ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                                ctypes.POINTER(ctypes.c_int32)])
_draw_samples = _sig("lmscale_draw_samples", _S, [_P, ctypes.c_uint64, ctypes.c_uint64, _i64, _P,
                                                  _P])
_lookup = _sig("lmscale_lookup", _S, [_P, _P, _i64, _P, _P, _P])
_set_codec = _sig("lmscale_set_codec", _S, [_P, ctypes.c_int32])
_set_compression = _sig("lmscale_set_compression", _S, [_P, ctypes.c_float])
_compress = _sig("lmscale_compress", _S, [_P, _P, _i64, ctypes.c_float, _P, _P])
_decompress = _sig("lmscale_decompress", _S, [_P, _P, _i64, ctypes.c_float, _P, _P])
_get_stats = _sig("lmscale_get_stats", _S, [_P, ctypes.POINTER(StatsC)])
_status_string = _sig("lmscale_status_string", ctypes.c_char_p, [_S])
_last_error = _sig("lmscale_last_error", ctypes.c_char_p, [_P])
_version = _sig("lmscale_version", ctypes.c_char_p, [])

EXPORTED = ["lmscale_get_nccl_id", "lmscale_init", "lmscale_destroy", "lmscale_unique",
            "lmscale_global_unique", "lmscale_scatter_expand", "lmscale_get_sparse_grad",
            "lmscale_get_local_maps", "lmscale_sync_embedding_grad",
            "lmscale_apply_sparse_update", "lmscale_step", "lmscale_emulate_step",
            "lmscale_sync_dense_baseline",
            "lmscale_dense_apply", "lmscale_train_step_host", "lmscale_set_timing", "lmscale_alloc_table",
            "lmscale_set_compression", "lmscale_set_codec", "lmscale_compress", "lmscale_decompress",
            "lmscale_plan_seeds", "lmscale_draw_samples", "lmscale_lookup", "lmscale_get_stats",
            "lmscale_status_string", "lmscale_last_error", "lmscale_version"]


SEED_POLICIES = {"distinct": 0, "same": 1, "log2": 2, "loge": 3, "log10": 4, "power": 5}


def plan_seeds(world: int, policy: str = "power", alpha: float = 0.64, master_seed: int = 0):
    """Sec. 3.2 seed groups (host only): (seeds per rank, number of groups)."""
    seeds = (ctypes.c_uint64 * world)()
    n = ctypes.c_int32()
    st = _plan_seeds(int(world), SEED_POLICIES[policy], float(alpha),
                     int(master_seed) & (2**64 - 1), seeds, ctypes.byref(n))
    if st != OK:
        raise LmscaleError(st, f"lmscale_plan_seeds({world}, {policy}, {alpha})")
    return [int(x) for x in seeds], int(n.value)


def emulate_step(ctxs, ids, grads, tables, lr, stream=None):
    """lmscale_emulate_step: the world-G step of lmscale_step on one GPU.
    ctxs[r] are NO_COMM contexts (world = len(ctxs), rank r); ids[r], grads[r]
    and tables[r] are rank r's device tensors (tables updated in place)."""
    G = len(ctxs)
    assert len(ids) == len(grads) == len(tables) == G
    ids = [Context._ids(t) for t in ids]
    k = ids[0].numel()
    for g, t, i in zip(grads, tables, ids):
        assert i.numel() == k
        assert g.dtype == torch.float32 and g.is_cuda and g.is_contiguous()
        assert t.dtype == torch.float32 and t.is_cuda and t.is_contiguous()
    arr = lambda xs: (_P * G)(*[_ptr(x) for x in xs])  # noqa: E731
    hs = (_P * G)(*[c._h for c in ctxs])
    st = _emulate_step(hs, G, arr(ids), arr(grads), k, arr(tables), float(lr), _stream(stream))
    if st != OK:
        raise LmscaleError(st, "lmscale_emulate_step: " + (_last_error(ctxs[0]._h) or b"").decode())


class LmscaleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_status_string(status).decode()} ({status}): {msg}")
        self.status = status


def version() -> str:
    return _version().decode()


def get_nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = _get_nccl_id(buf)
    if st != OK:
        raise LmscaleError(st, "ncclGetUniqueId")
    return buf.raw


class _DevArray:
    """Zero-copy __cuda_array_interface__ view of workspace memory."""

    def __init__(self, ptr, shape, typestr, device):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}
        self.device = device


def _view(ptr, shape, dtype, device):
    typestr = {torch.uint32: "<u4", torch.int32: "<i4", torch.float32: "<f4",
               torch.int16: "<i2"}[dtype]
    n = 1
    for s in shape:
        n *= s
    if n == 0 or not ptr:
        return torch.empty(shape, dtype=dtype, device=device)
    with torch.cuda.device(device):
        return torch.as_tensor(_DevArray(ptr, shape, typestr, device), device=device)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class SparseGrad:
    """I^ (uint32[U_g]), the global counts (int32[U_g], or None) and M^
    (float32[U_g, D], or None when a step consumed it) as zero-copy device views."""

    def __init__(self, c: SparseGradC, dim: int, device):
        self.c = c
        self.num_unique = int(c.num_unique)
        n = max(self.num_unique, 0)
        self.ids = _view(c.ids, (n,), torch.int32, device)  # uint32 bit patterns
        self.counts = _view(c.counts, (n,), torch.int32, device) if c.counts else None
        self.rows = _view(c.rows, (n, dim), torch.float32, device) if c.rows else None

    @classmethod
    def from_tensors(cls, ids: torch.Tensor, rows: torch.Tensor) -> "SparseGrad":
        """Wrap caller-owned I^ (uint32[U]) and rows (float32[U, D]) device tensors."""
        assert ids.is_cuda and rows.is_cuda and rows.is_contiguous() and ids.is_contiguous()
        assert rows.dtype == torch.float32 and ids.numel() == rows.shape[0]
        self = cls.__new__(cls)
        self.c = SparseGradC(ids.data_ptr(), None, rows.data_ptr(), ids.numel())
        self.num_unique = ids.numel()
        self.ids, self.rows, self.counts = ids, rows, None
        return self


class Context:
    """One rank of the exchange (lmscale_init / lmscale_destroy)."""

    def __init__(self, vocab, max_tokens, dim, world=1, rank=0, device=None, flags=0,
                 nccl_id: bytes | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.dim = int(dim)
        self.world = int(world)
        self.cfg = Config(int(vocab), int(max_tokens), int(dim), int(world), int(rank),
                          int(device), int(flags))
        h = _P()
        st = _init(ctypes.byref(self.cfg), nccl_id, ctypes.byref(h))
        if st != OK:
            raise LmscaleError(st, "lmscale_init")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != OK:
            raise LmscaleError(st, f"{what}: {_last_error(self._h).decode()}")

    @staticmethod
    def _ids(t):
        assert t.dtype in (torch.uint32, torch.int32) and t.is_cuda and t.is_contiguous()
        return t

    # ---- staged
    def unique(self, ids, want_outputs=True, stream=None):
        """S1: returns (J^ uint32[U_i], counts int32[U_i], inverse int32[K])."""
        ids = self._ids(ids)
        k = ids.numel()
        if want_outputs:
            uniq = torch.empty(k, dtype=torch.int32, device=ids.device)   # uint32 bit patterns
            counts = torch.empty(k, dtype=torch.int32, device=ids.device)
            inverse = torch.empty(k, dtype=torch.int32, device=ids.device)
            nu = torch.zeros(1, dtype=torch.int64, device=ids.device)
            self._check(_unique(self._h, _ptr(ids), k, _ptr(uniq), _ptr(counts), _ptr(inverse),
                                _ptr(nu), _stream(stream)), "lmscale_unique")
            u = int(nu.item())
            return uniq[:u], counts[:u], inverse
        self._check(_unique(self._h, _ptr(ids), k, None, None, None, None, _stream(stream)),
                    "lmscale_unique")
        return None

    def global_unique(self, gathered, stream=None):
        gathered = self._ids(gathered)
        self._check(_global_unique(self._h, _ptr(gathered), gathered.numel(), _stream(stream)),
                    "lmscale_global_unique")

    def scatter_expand(self, grad, stream=None):
        assert grad.dtype == torch.float32 and grad.is_cuda and grad.is_contiguous()
        self._check(_scatter_expand(self._h, _ptr(grad), grad.shape[0], _stream(stream)),
                    "lmscale_scatter_expand")

    def sparse_grad(self, stream=None) -> SparseGrad:
        c = SparseGradC()
        self._check(_get_sparse_grad(self._h, ctypes.byref(c), _stream(stream)),
                    "lmscale_get_sparse_grad")
        return SparseGrad(c, self.dim, self.device)

    def local_maps(self, stream=None):
        """(J^, counts, inverse, l2g) of the last S1/S3, as device views."""
        u, c, inv, l2g = _P(), _P(), _P(), _P()
        n = _i64()
        self._check(_get_local_maps(self._h, ctypes.byref(u), ctypes.byref(c), ctypes.byref(inv),
                                    ctypes.byref(l2g), ctypes.byref(n), _stream(stream)),
                    "lmscale_get_local_maps")
        U = int(n.value)
        k = self.cfg.max_tokens
        return (_view(u.value, (U,), torch.int32, self.device),
                _view(c.value, (U,), torch.int32, self.device),
                _view(inv.value, (k,), torch.int32, self.device),
                _view(l2g.value, (U,), torch.int32, self.device) if l2g.value else None)

    # ---- collective path
    def sync(self, ids, grad, stream=None) -> SparseGrad:
        """S1-S5: the uniqueness exchange; returns I^ and the all-reduced M^."""
        ids = self._ids(ids)
        assert grad.dtype == torch.float32 and grad.is_cuda and grad.is_contiguous()
        assert grad.shape == (ids.numel(), self.dim)
        c = SparseGradC()
        self._check(_sync(self._h, _ptr(ids), _ptr(grad), ids.numel(), ctypes.byref(c),
                          _stream(stream)), "lmscale_sync_embedding_grad")
        return SparseGrad(c, self.dim, self.device)

    def apply_update(self, table, sg: SparseGrad, lr: float, stream=None):
        """S6: table[I^[r]] -= lr * M^[r] (in place)."""
        assert table.dtype == torch.float32 and table.is_cuda and table.is_contiguous()
        self._check(_apply(self._h, _ptr(table), ctypes.byref(sg.c), float(lr), _stream(stream)),
                    "lmscale_apply_sparse_update")

    def step(self, ids, grad, table, lr, want_num_unique=False, stream=None):
        """S1-S6 in one C call (lmscale_step).  Returns U_g if asked (that
        forces a host sync), else None -- with world == 1 the call then
        returns as soon as the kernels are enqueued."""
        ids = self._ids(ids)
        assert grad.dtype == torch.float32 and grad.is_cuda and grad.is_contiguous()
        assert table.dtype == torch.float32 and table.is_cuda and table.is_contiguous()
        n = _i64(-1)
        self._check(_step(self._h, _ptr(ids), _ptr(grad), ids.numel(), _ptr(table), float(lr),
                          ctypes.byref(n) if want_num_unique else None, _stream(stream)),
                    "lmscale_step")
        return int(n.value) if want_num_unique else None

    def sync_dense(self, ids, grad, table, lr, stream=None):
        """S0: dense all-gather baseline, table updated in place."""
        ids = self._ids(ids)
        self._check(_dense(self._h, _ptr(ids), _ptr(grad), ids.numel(), _ptr(table), float(lr),
                           _stream(stream)), "lmscale_sync_dense_baseline")

    def dense_apply(self, ids, grad, table, lr, stream=None):
        ids = self._ids(ids)
        self._check(_dense_apply(self._h, _ptr(ids), _ptr(grad), ids.numel(), _ptr(table),
                                 float(lr), _stream(stream)), "lmscale_dense_apply")

    def train_step_host(self, ids_host, grad_host, table, lr, ids_out_host=None, stream=None):
        """End-to-end step from host (pinned) buffers; returns U_g."""
        assert not ids_host.is_cuda and not grad_host.is_cuda
        n = _i64()
        self._check(_host_step(self._h, _ptr(ids_host), _ptr(grad_host), ids_host.numel(),
                               _ptr(table), float(lr), _ptr(ids_out_host), ctypes.byref(n),
                               _stream(stream)), "lmscale_train_step_host")
        return int(n.value)

    def alloc_table(self) -> torch.Tensor:
        """The context-owned vocab x dim table (lmscale_alloc_table): with world > 1
        and NVLS it is a symmetric window and updates are multicast into every
        replica.  Collective when world > 1.  Returns a zero-copy float32 view."""
        p, n = _P(), _i64()
        self._check(_alloc_table(self._h, ctypes.byref(p), ctypes.byref(n)), "lmscale_alloc_table")
        return _view(p.value, (int(self.cfg.vocab), self.dim), torch.float32, self.device)

    def set_timing(self, mode: int):
        """0 none, 1 S4-only events, 2 every phase (see lmscale_set_timing)."""
        self._check(_set_timing(self._h, int(mode)), "lmscale_set_timing")

    def set_compression(self, F: float):
        """Sec. 3.3 compressed exchange for later collective steps; 0 = off."""
        self._check(_set_compression(self._h, float(F)), "lmscale_set_compression")

    def set_codec(self, codec: str):
        """16-bit payload format: "fp16" (binary16, default) or "bf16"."""
        self._check(_set_codec(self._h, {"fp16": 0, "bf16": 1}[codec]), "lmscale_set_codec")

    def compress(self, x, F, stream=None) -> torch.Tensor:
        """binary16 bits (as int16) of RNE(fp32(F * x)), saturated."""
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        q = torch.empty(x.shape, dtype=torch.int16, device=x.device)
        self._check(_compress(self._h, _ptr(x), x.numel(), float(F), _ptr(q), _stream(stream)),
                    "lmscale_compress")
        return q

    def decompress(self, q, F, stream=None) -> torch.Tensor:
        """fp32(q) / F; q holds binary16 bits (int16 or float16 tensor)."""
        assert q.is_cuda and q.element_size() == 2 and q.is_contiguous()
        x = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        self._check(_decompress(self._h, _ptr(q), q.numel(), float(F), _ptr(x), _stream(stream)),
                    "lmscale_decompress")
        return x

    def draw_samples(self, seed: int, step: int, S: int, out=None, stream=None) -> torch.Tensor:
        """Sec. 3.2 candidates: S distinct ids of the (seed, step) stream (R16),
        as an int32 view of the uint32 ids; written into `out` when given."""
        if out is None:
            out = torch.empty(S, dtype=torch.int32, device=self.device)
        assert out.is_cuda and out.numel() >= S and out.element_size() == 4 and out.is_contiguous()
        self._check(_draw_samples(self._h, int(seed) & (2**64 - 1), int(step) & (2**64 - 1), int(S),
                                  _ptr(out), _stream(stream)), "lmscale_draw_samples")
        return out[:S]

    def lookup(self, ids, table, out=None, stream=None) -> torch.Tensor:
        """Forward lookup out[p] = table[ids[p]]."""
        ids = self._ids(ids)
        if out is None:
            out = torch.empty(ids.numel(), self.dim, dtype=torch.float32, device=self.device)
        self._check(_lookup(self._h, _ptr(ids), ids.numel(), _ptr(table), _ptr(out),
                            _stream(stream)), "lmscale_lookup")
        return out

    def stats(self) -> dict:
        s = StatsC()
        self._check(_get_stats(self._h, ctypes.byref(s)), "lmscale_get_stats")
        return {f: getattr(s, f) for f, _ in StatsC._fields_}
