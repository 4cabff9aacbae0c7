"""CPU oracle for the uniqueness embedding-gradient exchange (arXiv 1810.10045 Sec. 3.1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1810_10045_b200`` never imports it, and
the two share no code.

The arithmetic lives in ``oracle.c`` (plain loops, fp64 accumulation, one
rounding to fp32).  This module only marshals numpy arrays through ctypes and
strings the paper's seven steps together in the paper's order:

1. local unique J^          -> ``unique_local``
2. local reduction Delta^   -> ``reduce_local``
3. AllGather of J -> I      -> ``allgather_ids``
4. global unique I^ + maps  -> ``unique_global``, ``remap``
5. expand to M_i, zeros     -> ``scatter_expand``
6. AllReduce -> M^          -> ``allreduce_sum``
7. row update of E          -> ``update_rows``

``sync_unique`` runs the seven steps for G simulated ranks; ``sync_dense``
is the baseline all-gather exchange.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no fast-math: fp64 stays IEEE)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64 = ctypes.c_int64
            lib.oracle_unique_local.restype = i64
            lib.oracle_unique_local.argtypes = [P, i64, P, P, P]
            lib.oracle_reduce_local.restype = None
            lib.oracle_reduce_local.argtypes = [P, i64, i64, P, i64, P]
            lib.oracle_reduce_local_cols.restype = None
            lib.oracle_reduce_local_cols.argtypes = [P, i64, i64, P, i64, P, i64, i64]
            lib.oracle_allgather_ids.restype = None
            lib.oracle_allgather_ids.argtypes = [P, P, ctypes.c_int, P]
            lib.oracle_unique_global.restype = i64
            lib.oracle_unique_global.argtypes = [P, i64, P, P]
            lib.oracle_remap.restype = None
            lib.oracle_remap.argtypes = [P, i64, P, i64, P, i64, P, P]
            lib.oracle_scatter_expand.restype = None
            lib.oracle_scatter_expand.argtypes = [P, i64, i64, P, i64, P]
            lib.oracle_allreduce_sum.restype = None
            lib.oracle_allreduce_sum.argtypes = [P, ctypes.c_int, i64, P]
            lib.oracle_update_rows.restype = None
            lib.oracle_update_rows.argtypes = [P, i64, P, i64, P, ctypes.c_double]
            lib.oracle_sync_dense.restype = None
            lib.oracle_sync_dense.argtypes = [P, P, i64, i64, ctypes.c_int, P, P, P,
                                              ctypes.c_double]
            lib.oracle_type_gradient.restype = i64
            lib.oracle_compress.restype = None
            lib.oracle_compress.argtypes = [P, i64, ctypes.c_float, P]
            lib.oracle_decompress.restype = None
            lib.oracle_decompress.argtypes = [P, i64, ctypes.c_float, P]
            lib.oracle_compress_bf16.restype = None
            lib.oracle_compress_bf16.argtypes = [P, i64, ctypes.c_float, P]
            lib.oracle_decompress_bf16.restype = None
            lib.oracle_decompress_bf16.argtypes = [P, i64, ctypes.c_float, P]
            lib.oracle_sum_f32.restype = None
            lib.oracle_sum_f32.argtypes = [P, ctypes.c_int, i64, P]
            lib.oracle_mix64.restype = ctypes.c_uint64
            lib.oracle_mix64.argtypes = [ctypes.c_uint64]
            lib.oracle_draw_one.restype = ctypes.c_uint32
            lib.oracle_draw_one.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64]
            lib.oracle_draw_samples.restype = i64
            lib.oracle_draw_samples.argtypes = [ctypes.c_uint64, ctypes.c_uint64, i64,
                                                ctypes.c_uint64, P]
            lib.oracle_lookup.restype = None
            lib.oracle_lookup.argtypes = [P, i64, i64, P, i64, P]
            lib.oracle_type_gradient.argtypes = [P, P, P, ctypes.c_int, i64,
                                                 ctypes.c_uint32, P, P]
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr_array(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


# --------------------------------------------------------------------------- steps

def unique_local(J):
    """Step 1. Returns (J^ ascending uint32, counts int32, inverse int32)."""
    lib = _load()
    J = _u32(J)
    K = J.size
    uniq = np.empty(K, np.uint32)
    counts = np.empty(K, np.int32)
    inverse = np.empty(K, np.int32)
    U = lib.oracle_unique_local(_p(J), K, _p(uniq), _p(counts), _p(inverse))
    return uniq[:U].copy(), counts[:U].copy(), inverse


def reduce_local(delta, inverse, U):
    """Step 2. fp64 Delta^ (U x D), ascending-position sums."""
    lib = _load()
    delta = _f32(delta)
    K, D = delta.shape
    inverse = np.ascontiguousarray(inverse, dtype=np.int32)
    out = np.empty((U, D), np.float64)
    lib.oracle_reduce_local(_p(delta), K, D, _p(inverse), U, _p(out))
    return out


def reduce_local_threads(delta, inverse, U, threads):
    """Step 2 split over ``threads`` column blocks run concurrently (ctypes
    releases the GIL): bit-identical to ``reduce_local`` (same loop, same
    per-element order).  bench.py's all-cores cpu_baseline only."""
    from concurrent.futures import ThreadPoolExecutor
    lib = _load()
    delta = _f32(delta)
    K, D = delta.shape
    inverse = np.ascontiguousarray(inverse, dtype=np.int32)
    out = np.empty((U, D), np.float64)
    nt = max(1, min(int(threads), D))
    cuts = [D * t // nt for t in range(nt + 1)]
    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(lambda t: lib.oracle_reduce_local_cols(_p(delta), K, D, _p(inverse), U,
                                                           _p(out), cuts[t], cuts[t + 1]),
                    range(nt)))
    return out


def allgather_ids(J_list):
    """Step 3. Rank-ordered concatenation I of every rank's J."""
    lib = _load()
    Js = [_u32(j) for j in J_list]
    Ks = np.array([j.size for j in Js], np.int64)
    I = np.empty(int(Ks.sum()), np.uint32)
    lib.oracle_allgather_ids(_ptr_array(Js), _p(Ks), len(Js), _p(I))
    return I


def unique_global(I):
    """Step 4. Returns (I^ ascending uint32, global counts int32)."""
    lib = _load()
    I = _u32(I)
    n = I.size
    Ihat = np.empty(n, np.uint32)
    gcounts = np.empty(n, np.int32)
    U = lib.oracle_unique_global(_p(I), n, _p(Ihat), _p(gcounts))
    return Ihat[:U].copy(), gcounts[:U].copy()


def remap(Jhat, Ihat, inverse):
    """Step 4 maps: l2g (J^ -> I^) and slot (J -> I^)."""
    lib = _load()
    Jhat = _u32(Jhat)
    Ihat = _u32(Ihat)
    inverse = np.ascontiguousarray(inverse, dtype=np.int32)
    l2g = np.empty(Jhat.size, np.int32)
    slot = np.empty(inverse.size, np.int32)
    lib.oracle_remap(_p(Jhat), Jhat.size, _p(Ihat), Ihat.size, _p(inverse),
                     inverse.size, _p(l2g), _p(slot))
    return l2g, slot


def scatter_expand(dhat, l2g, Ug):
    """Step 5. fp64 M_i (Ug x D): Delta^ rows at l2g, zeros elsewhere."""
    lib = _load()
    dhat = np.ascontiguousarray(dhat, dtype=np.float64)
    Ui, D = dhat.shape
    l2g = np.ascontiguousarray(l2g, dtype=np.int32)
    M = np.empty((Ug, D), np.float64)
    lib.oracle_scatter_expand(_p(dhat), Ui, D, _p(l2g), Ug, _p(M))
    return M


def allreduce_sum(M_list):
    """Step 6. Rank-ordered fp64 sum of the M_i."""
    lib = _load()
    Ms = [np.ascontiguousarray(m, dtype=np.float64) for m in M_list]
    out = np.empty_like(Ms[0])
    lib.oracle_allreduce_sum(_ptr_array(Ms), len(Ms), out.size, _p(out))
    return out


def update_rows(E, Ihat, Mhat64, lr):
    """Step 7. In place: E[I^[r]] = round32(E[I^[r]] - lr * M^64[r])."""
    lib = _load()
    assert E.dtype == np.float32 and E.flags.c_contiguous
    Ihat = _u32(Ihat)
    Mhat64 = np.ascontiguousarray(Mhat64, dtype=np.float64)
    D = E.shape[1]
    lib.oracle_update_rows(_p(E), D, _p(Ihat), Ihat.size, _p(Mhat64), float(lr))
    return E


# ---------------------------------------------------------------- composites

def sync_unique(J_list, delta_list, E, lr):
    """The uniqueness exchange, steps 1-7 for G simulated ranks.

    ``E`` (V x D fp32) is updated in place (one replica stands for all G:
    they receive the same M^ and I^).  Returns a dict of every intermediate.
    """
    G = len(J_list)
    ranks = []
    for g in range(G):                                   # steps 1, 2
        Jhat, counts, inverse = unique_local(J_list[g])
        dhat = reduce_local(delta_list[g], inverse, Jhat.size)
        ranks.append(dict(Jhat=Jhat, counts=counts, inverse=inverse, dhat=dhat))
    I = allgather_ids(J_list)                            # step 3
    Ihat, gcounts = unique_global(I)                     # step 4
    Ug = Ihat.size
    Ms = []
    for r in ranks:
        r["l2g"], r["slot"] = remap(r["Jhat"], Ihat, r["inverse"])
        Ms.append(scatter_expand(r["dhat"], r["l2g"], Ug))   # step 5
    Mhat64 = allreduce_sum(Ms)                           # step 6
    update_rows(E, Ihat, Mhat64, lr)                     # step 7
    return dict(ranks=ranks, I=I, Ihat=Ihat, Ug=Ug, gcounts=gcounts, M=Ms,
                Mhat64=Mhat64, Mhat=Mhat64.astype(np.float32), E=E)


def sync_unique_threads(J_list, delta_list, E, lr, threads):
    """``sync_unique`` with step 2 (the Theta(KD) local reduction, the bulk of
    the work) split over ``threads`` column blocks: the same seven steps in
    the same order, bit-identical results (bench.py's all-cores cpu_baseline)."""
    G = len(J_list)
    ranks = []
    for g in range(G):                                   # steps 1, 2
        Jhat, counts, inverse = unique_local(J_list[g])
        dhat = reduce_local_threads(delta_list[g], inverse, Jhat.size, threads)
        ranks.append(dict(Jhat=Jhat, counts=counts, inverse=inverse, dhat=dhat))
    I = allgather_ids(J_list)                            # step 3
    Ihat, gcounts = unique_global(I)                     # step 4
    Ug = Ihat.size
    Ms = []
    for r in ranks:
        r["l2g"], r["slot"] = remap(r["Jhat"], Ihat, r["inverse"])
        Ms.append(scatter_expand(r["dhat"], r["l2g"], Ug))   # step 5
    Mhat64 = allreduce_sum(Ms)                           # step 6
    update_rows(E, Ihat, Mhat64, lr)                     # step 7
    return dict(ranks=ranks, I=I, Ihat=Ihat, Ug=Ug, gcounts=gcounts, M=Ms,
                Mhat64=Mhat64, Mhat=Mhat64.astype(np.float32), E=E)


def compress(x, F, fmt="fp16"):
    """Sec. 3.3: 16-bit payload (uint16 bits) of RNE(fp32(F * x)),
    saturated to the format's largest finite value (R15);
    fmt = "fp16" (binary16, the paper's) or "bf16"."""
    lib = _load()
    x = _f32(x)
    q = np.empty(x.shape, np.uint16)
    fn = lib.oracle_compress if fmt == "fp16" else lib.oracle_compress_bf16
    fn(_p(x), x.size, float(F), _p(q))
    return q


def decompress(q, F, fmt="fp16"):
    """Sec. 3.3: fp32(payload) / F."""
    lib = _load()
    q = np.ascontiguousarray(q, dtype=np.uint16)
    x = np.empty(q.shape, np.float32)
    fn = lib.oracle_decompress if fmt == "fp16" else lib.oracle_decompress_bf16
    fn(_p(q), q.size, float(F), _p(x))
    return x


def sum_f32(a_list):
    """Rank-ordered fp32 sum of the up-cast payloads (R15)."""
    lib = _load()
    As = [_f32(a) for a in a_list]
    out = np.empty_like(As[0])
    lib.oracle_sum_f32(_ptr_array(As), len(As), out.size, _p(out))
    return out


def sync_unique_compressed(J_list, delta_list, E, lr, F, fmt="fp16"):
    """The uniqueness exchange with compression (Sec. 3.3 on Sec. 3.1).

    Steps 1-5 as ``sync_unique``; each M_i is an FP32 tensor, so it is
    rounded once to fp32.  Step 6, the all-reduce, runs as the two exchanges
    of a reduce-scatter + all-gather, each with the paper's codec (R15):

    a. every rank sends compress(M_i, F); the receiver up-casts, divides by F
       and sums in fp32, rank order -> S;
    b. S is sent as compress(S, F) and every rank up-casts and divides:
       M^ = decompress(compress(S, F), F).

    Step 7 is ``update_rows`` with that M^.  E is updated in place.
    """
    G = len(J_list)
    ranks = []
    for g in range(G):                                   # steps 1, 2
        Jhat, counts, inverse = unique_local(J_list[g])
        dhat = reduce_local(delta_list[g], inverse, Jhat.size)
        ranks.append(dict(Jhat=Jhat, counts=counts, inverse=inverse, dhat=dhat))
    I = allgather_ids(J_list)                            # step 3
    Ihat, gcounts = unique_global(I)                     # step 4
    Ug = Ihat.size
    M32, Q = [], []
    for r in ranks:
        r["l2g"], r["slot"] = remap(r["Jhat"], Ihat, r["inverse"])
        m = scatter_expand(r["dhat"], r["l2g"], Ug).astype(np.float32)   # step 5
        M32.append(m)
        Q.append(compress(m, F, fmt))                    # 6a: down-cast on the sender
    S = sum_f32([decompress(q, F, fmt) for q in Q])      # 6a: up-cast, sum (receiver)
    Qhat = compress(S, F, fmt)                           # 6b: the reduced rows, down-cast
    Mhat = decompress(Qhat, F, fmt)                      # 6b: up-cast on every rank
    update_rows(E, Ihat, Mhat.astype(np.float64), lr)    # step 7
    return dict(ranks=ranks, I=I, Ihat=Ihat, Ug=Ug, gcounts=gcounts, M32=M32, Q=Q, S=S,
                Qhat=Qhat, Mhat=Mhat, E=E)


def lookup(E, J):
    """Forward lookup: out[p] = E[J[p]] (zero row for J[p] >= V)."""
    lib = _load()
    E = _f32(E)
    J = _u32(J)
    V, D = E.shape
    out = np.empty((J.size, D), np.float32)
    lib.oracle_lookup(_p(E), V, D, _p(J), J.size, _p(out))
    return out


# ------------------------------------------------------------ seeding (3.2)

SEED_POLICIES = ("distinct", "same", "log2", "loge", "log10", "power")


def plan_seeds(G, policy, alpha=0.64, master_seed=0):
    """Seed groups of Sec. 3.2 (R16): "make a subset of GPUs use the
    same seed"; policies all-distinct, all-same, log2/ln/log10 of G ("number of
    seeds equal to log2, loge, and log10 of the number of GPUs") and
    G^alpha ("we only need G^alpha unique random seeds").  Group counts
    as SPEC S:325: log_b -> max(1, round(log_b G)), power -> max(1, ceil(G^a)).
    Ranks go to groups in contiguous blocks: group(r) = floor(r * n / G).
    Seed of group q = mix64(master_seed + q).  Returns (seeds[G], n_groups)."""
    import math
    if policy == "distinct":
        n = G
    elif policy == "same":
        n = 1
    elif policy in ("log2", "loge", "log10"):
        b = {"log2": 2.0, "loge": math.e, "log10": 10.0}[policy]
        n = max(1, int(math.floor(math.log(G) / math.log(b) + 0.5)))
    elif policy == "power":
        if not (0.0 < alpha <= 1.0):
            raise ValueError("alpha must be in (0, 1]")
        n = max(1, int(math.ceil(G ** alpha)))
    else:
        raise ValueError(policy)
    n = min(n, G)
    lib = _load()
    seeds = [int(lib.oracle_mix64((master_seed + (r * n) // G) & (2**64 - 1))) for r in range(G)]
    return seeds, n


def draw_samples(seed, step, S, V):
    """The first S distinct values of the R16 stream, in stream order (uint32)."""
    if S > V:
        raise ValueError("S > V")
    lib = _load()
    out = np.empty(S, np.uint32)
    lib.oracle_draw_samples(seed & (2**64 - 1), step & (2**64 - 1), S, V, _p(out))
    return out


def draw_one(seed, step, i, V):
    return int(_load().oracle_draw_one(seed, step, i, V))


def mix64(z):
    return int(_load().oracle_mix64(z & (2**64 - 1)))


def sync_dense(J_list, delta_list, E, lr):
    """Baseline all-gather exchange; E (V x D fp32) updated in place."""
    lib = _load()
    assert E.dtype == np.float32 and E.flags.c_contiguous
    V, D = E.shape
    Js = [_u32(j) for j in J_list]
    Ds = [_f32(d) for d in delta_list]
    Ks = np.array([j.size for j in Js], np.int64)
    E64 = np.empty((V, D), np.float64)
    lib.oracle_sync_dense(_p(E), _p(E64), V, D, len(Js), _ptr_array(Js), _ptr_array(Ds),
                          _p(Ks), float(lr))
    return E


def type_gradient(J_list, delta_list, w):
    """One row of M^ from the definition: fp64 sum of every Delta row of
    word ``w`` over all ranks, plus the summation-error scale A = sum |Delta|.
    Returns (row fp64[D], A fp64[D], number of tokens)."""
    lib = _load()
    Js = [_u32(j) for j in J_list]
    Ds = [_f32(d) for d in delta_list]
    Ks = np.array([j.size for j in Js], np.int64)
    D = Ds[0].shape[1]
    out = np.empty(D, np.float64)
    absout = np.empty(D, np.float64)
    n = lib.oracle_type_gradient(_ptr_array(Js), _ptr_array(Ds), _p(Ks), len(Js), D,
                                 int(w), _p(out), _p(absout))
    return out, absout, int(n)


def abs_scale(J_list, delta_list, Ihat):
    """A[r,:] = sum of |Delta| over every token of word I^[r] (fp64) -- the
    summation-error scale of the SIGNED-mode metric.
    Same loop as steps 1-6 applied to |Delta|."""
    absd = [np.abs(_f32(d)) for d in delta_list]
    Ms = []
    for J, a in zip(J_list, absd):
        Jhat, _, inverse = unique_local(J)
        dh = reduce_local(a, inverse, Jhat.size)
        l2g, _ = remap(Jhat, Ihat, inverse)
        Ms.append(scatter_expand(dh, l2g, len(Ihat)))
    return allreduce_sum(Ms)


def complexity_plan(G, K, D, alpha, elem_bytes=4, index_bytes=4):
    """Sec. 3.1 complexity: dense Theta(GKD) bytes vs
    unique Theta(GK + U_g D) with U_g estimated as (GK)^alpha."""
    baseline = G * K * D * elem_bytes
    ug = (G * K) ** alpha
    grad = ug * D * elem_bytes
    idx = G * K * index_bytes
    return dict(baseline_bytes=baseline, u_g_estimate=ug, unique_grad_bytes=grad,
                unique_index_bytes=idx, saving_factor=baseline / (idx + grad),
                saving_factor_grad_only=baseline / grad)
