"""Pins for the compression oracle (Sec. 3.3; R15).

The codec is pinned by the SPEC's worked values and hand-written IEEE-754
binary16 bit patterns (tests/golden/compression.json), by numpy's own
float32 -> float16 conversion (a library routine, round-to-nearest-even), by
the exhaustive round trip of every finite binary16 value, and by the unit
roundoff bound.  The compressed exchange is pinned by the special case that
reduces to the uncompressed exchange (every payload exactly representable)
and by its error bound against the fp64 exchange.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _np_half(x, F):
    """numpy's binary16 RNE of fp32(F * x), saturated (R15)."""
    p = (np.float32(F) * np.asarray(x, np.float32)).astype(np.float32)
    p = np.clip(p, np.float32(-65504.0), np.float32(65504.0))
    return p.astype(np.float16).view(np.uint16)


def test_golden_values():
    g = json.load(open(os.path.join(GOLD, "compression.json")))
    for c in g["cases"]:
        q = oracle.compress(np.array([c["x"]], np.float32), c["F"])
        assert int(q[0]) == c["bits"], c["cite"]
        back = oracle.decompress(q, c["F"])
        assert back[0] == np.float32(c["back"]), c["cite"]


def test_payload_is_half_the_bytes():
    x = np.linspace(-3, 3, 1001, dtype=np.float32)
    q = oracle.compress(x, 256.0)
    assert q.nbytes * 2 == x.nbytes            # "reduces the communication by 50%"


def test_every_finite_half_round_trips():
    bits = np.arange(1 << 16, dtype=np.uint16)
    h = bits.view(np.float16)
    finite = np.isfinite(h)
    bits = bits[finite]
    x = oracle.decompress(bits, 1.0)
    np.testing.assert_array_equal(x, bits.view(np.float16).astype(np.float32))  # exact widening
    np.testing.assert_array_equal(oracle.compress(x, 1.0), bits)                # bijection


@pytest.mark.parametrize("F", [1.0, 256.0, 512.0, 1024.0, 3.0])
def test_compress_matches_numpy_rne(F):
    rng = np.random.default_rng(1810)
    x = np.concatenate([
        rng.standard_normal(20000).astype(np.float32),
        (rng.standard_normal(20000) * 1e-6).astype(np.float32),     # subnormal range
        (rng.standard_normal(5000) * 1e5).astype(np.float32),       # saturation range
        (rng.integers(-4096, 4096, 5000)).astype(np.float32),       # integer ties
        (rng.integers(-4096, 4096, 5000) + 0.5).astype(np.float32),
    ])
    np.testing.assert_array_equal(oracle.compress(x, F), _np_half(x, F))


def test_relative_error_in_normal_range():
    rng = np.random.default_rng(7)
    x = np.exp2(rng.uniform(-10, 10, 200000)).astype(np.float32) * rng.choice([-1, 1], 200000)
    x = x.astype(np.float32)
    back = oracle.decompress(oracle.compress(x, 1.0), 1.0).astype(np.float64)
    rel = np.abs(back - x) / np.abs(x)
    assert rel.max() <= 2.0 ** -11            # unit roundoff of binary16 (S:448 allows 2^-10)


def test_scaling_rescues_small_values():
    """compression-scaling keeps small gradients from becoming zero;
    monotone in F while nothing saturates."""
    x = np.full(1000, 2.0 ** -25, np.float32)
    assert np.count_nonzero(oracle.compress(x, 1.0)) == 0
    assert np.count_nonzero(oracle.compress(x, 1024.0)) == 1000
    rng = np.random.default_rng(3)
    y = (rng.standard_normal(5000) * 1e-6).astype(np.float32)
    flushed = [np.count_nonzero((oracle.compress(y, F) & 0x7FFF) == 0) for F in (1, 4, 64, 1024)]
    assert flushed == sorted(flushed, reverse=True) and flushed[-1] < flushed[0]


# ------------------------------------------------------------ the exchange

def _tiny_ints(G, V=50, K=64, D=8, seed=0):
    rng = np.random.default_rng(seed)
    J = [rng.integers(0, V, K).astype(np.uint32) for _ in range(G)]
    Dl = [rng.integers(-8, 8, (K, D)).astype(np.float32) for _ in range(G)]
    E0 = (rng.integers(-16, 16, (V, D)) / 16).astype(np.float32)
    return J, Dl, E0


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("F", [1.0, 2.0])
def test_exchange_reduces_to_plain_when_exact(G, F):
    """Every payload an integer of magnitude <= 2048/F: the codec is the
    identity and the compressed exchange must equal the plain one bit for bit."""
    J, Dl, E0 = _tiny_ints(G)
    lr = 2.0 ** -4
    Ep = E0.copy()
    ref = oracle.sync_unique(J, Dl, Ep, lr)
    assert np.abs(ref["Mhat64"]).max() * F <= 2048
    Ec = E0.copy()
    got = oracle.sync_unique_compressed(J, Dl, Ec, lr, F)
    np.testing.assert_array_equal(got["Ihat"], ref["Ihat"])
    np.testing.assert_array_equal(got["Mhat"], ref["Mhat64"].astype(np.float32))
    np.testing.assert_array_equal(Ec, Ep)


def test_exchange_rounds_when_not_exact():
    """Large integer sums (> 2048) are not representable: the codec must round
    them (so a codec-free implementation fails this pin)."""
    G = 2
    J = [np.zeros(600, np.uint32) for _ in range(G)]
    Dl = [np.full((600, 2), 7.0, np.float32) for _ in range(G)]
    E0 = np.zeros((4, 2), np.float32)
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 1.0, 1.0)
    # each rank: 4200 -> binary16 ulp 4 at [4096, 8192): 4200 exactly; sum 8400
    # -> ulp 8 in [8192, 16384): 8400 = 8192 + 26*8 exactly representable
    assert got["Mhat"][0, 0] == 8400.0
    Dl = [np.full((601, 2), 7.0, np.float32) for _ in range(G)]
    J = [np.zeros(601, np.uint32) for _ in range(G)]
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 1.0, 1.0)
    # 4207 -> 4208 (ulp 4, RNE); 8416 = 8192 + 28*8 representable
    assert got["Mhat"][0, 0] == 8416.0


def test_exchange_codec_on_each_transfer_discriminates():
    """R15's reading -- the codec on each of the two transfers (sender payload,
    then the owner's reduced row) -- against a codec applied once to the exact
    sum: G = 2, one word, rank 0 contributes 2049, rank 1 contributes 1, F = 1.
    Two-stage: 2049 -> 2048 (binary16 RNE, tie to even), 1 -> 1, fp32 sum
    2049 -> 2048.  Single-stage would give compress(2050) = 2050.  A dropped
    sender-side codec would also give 2050; a ring that re-rounds partial
    sums hop by hop is not what the exchange does (R15)."""
    J = [np.array([3], np.uint32), np.array([3], np.uint32)]
    Dl = [np.array([[2049.0]], np.float32), np.array([[1.0]], np.float32)]
    E0 = np.zeros((5, 1), np.float32)
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 1.0, 1.0)
    assert got["Q"][0][0, 0] == np.float16(2048.0).view(np.uint16)     # sender rounding
    assert got["S"][0, 0] == 2049.0                                     # fp32 owner sum
    assert got["Mhat"][0, 0] == 2048.0                                  # second rounding
    assert got["E"][3, 0] == -2048.0
    plain = oracle.sync_unique(J, Dl, E0.copy(), 1.0)
    assert plain["Mhat64"][0, 0] == 2050.0
    single = oracle.decompress(oracle.compress(np.float32([2050.0]), 1.0), 1.0)
    assert single[0] == 2050.0 != got["Mhat"][0, 0]


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("F", [1.0, 32.0])
def test_exchange_error_bound_signed(G, F):
    """|M^c - M^| <= 2^-10 (sum_g |M_g| + |M^|) + (G+1) 2^-24 / F against the
    fp64 exchange: one binary16 rounding per payload element (<= 2^-11 relative,
    or half a subnormal ulp 2^-25/F absolute) on each of the two exchanges,
    plus fp32 roundings (2^-24)."""
    cfg = synth.CONFIGS["tiny"].with_(G=G)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dl = [synth.grad_values(cfg.K, cfg.D, "signed", rank=g).numpy() for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, "signed").numpy()
    ref = oracle.sync_unique(J, Dl, E0.copy(), 0.1)
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 0.1, F)
    assert np.abs(ref["Mhat64"]).max() * F < 65504            # no saturation
    absM = sum(np.abs(m) for m in ref["M"])
    bound = 2.0 ** -10 * (absM + np.abs(ref["Mhat64"])) + (G + 1) * 2.0 ** -24 / F
    err = np.abs(got["Mhat"].astype(np.float64) - ref["Mhat64"])
    assert (err <= bound).all()
    assert err.max() > 0                       # the codec did round something
    # dropping one rank's payload breaks the bound
    assert not (np.abs(got["Mhat"] - got["M32"][0] - ref["Mhat64"]) <= bound).all()


def test_exchange_saturates():
    """F * |M| beyond the binary16 range saturates: the reduced row is
    +-65504 / F, never inf."""
    G = 2
    J = [np.zeros(100, np.uint32) for _ in range(G)]
    Dl = [np.full((100, 3), 1.0, np.float32) for _ in range(G)]
    Dl[1][:, 1] = -1.0
    Dl[1][:, 2] = 0.0
    got = oracle.sync_unique_compressed(J, Dl, np.zeros((2, 3), np.float32), 1.0, 1024.0)
    # col 0: 100 -> 102400 saturates to 65504 on each rank, sum 131008 -> 65504
    # col 1: 65504 - 65504 = 0; col 2: 65504 + 0
    np.testing.assert_array_equal(got["Mhat"][0], np.float32([65504, 0, 65504]) / 1024)


# ------------------------------------------------------------ bfloat16 variant

def _torch_bf16(x, F):
    """torch's float32 -> bfloat16 (round to nearest even) of fp32(F * x),
    saturated to the largest finite bfloat16 (R15)."""
    import torch
    p = (np.float32(F) * np.asarray(x, np.float32)).astype(np.float32)
    m = np.float32(3.3895313892515355e38)
    p = np.clip(p, -m, m)
    return torch.from_numpy(p).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def test_bf16_golden_values():
    """Hand-written bfloat16 encodings: 1.0 = 0x3F80; 1 + 2^-8 is a tie -> even
    0x3F80; 1 + 3*2^-8 is a tie between 1 + 2^-7 and 1 + 2^-6 -> even 0x3F82
    (= 1 + 2^-6); -2 = 0xC000; saturation to 0x7F7F / 0xFF7F."""
    x = np.float32([1.0, 1 + 2**-8, 1 + 3 * 2**-8, -2.0, 3.4e38, -3.4e38, 0.0])
    want = [0x3F80, 0x3F80, 0x3F82, 0xC000, 0x7F7F, 0xFF7F, 0x0000]
    assert oracle.compress(x, 1.0, "bf16").tolist() == want
    back = oracle.decompress(np.uint16(want), 1.0, "bf16")
    assert back[0] == 1.0 and back[2] == np.float32(1 + 2**-6) and back[3] == -2.0


@pytest.mark.parametrize("F", [1.0, 3.0, 1024.0])
def test_bf16_matches_torch_rne(F):
    rng = np.random.default_rng(int(F) + 11)
    x = np.concatenate([
        rng.standard_normal(50000).astype(np.float32),
        (rng.standard_normal(20000) * 1e-38).astype(np.float32),     # subnormal range
        (rng.standard_normal(5000) * 1e36).astype(np.float32),
        rng.integers(-70000, 70000, 20000).astype(np.float32),       # ties
    ])
    np.testing.assert_array_equal(oracle.compress(x, F, "bf16"), _torch_bf16(x, F))


def test_bf16_round_trip_and_error():
    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    vals = (bits.astype(np.uint32) << 16).view(np.float32)
    finite = np.isfinite(vals)
    np.testing.assert_array_equal(oracle.compress(vals[finite], 1.0, "bf16"), bits[finite])
    np.testing.assert_array_equal(oracle.decompress(bits[finite], 1.0, "bf16"), vals[finite])
    rng = np.random.default_rng(5)
    x = (np.exp2(rng.uniform(-100, 100, 100000)) * rng.choice([-1, 1], 100000)).astype(np.float32)
    back = oracle.decompress(oracle.compress(x, 1.0, "bf16"), 1.0, "bf16").astype(np.float64)
    assert (np.abs(back - x) / np.abs(x)).max() <= 2.0 ** -8


@pytest.mark.parametrize("G", [2, 4])
def test_bf16_exchange_exact_case_and_bound(G):
    """Integers <= 256 are exact in bfloat16: the bf16 exchange equals the
    plain one; in SIGNED mode it stays within 2^-7 (sum|M_g| + |M^|)."""
    rng = np.random.default_rng(G)
    J = [rng.integers(0, 40, 16).astype(np.uint32) for _ in range(G)]
    Dl = [rng.integers(-4, 4, (16, 4)).astype(np.float32) for _ in range(G)]
    E0 = (rng.integers(-16, 16, (40, 4)) / 16).astype(np.float32)
    ref = oracle.sync_unique(J, Dl, E0.copy(), 2.0 ** -4)
    assert np.abs(ref["Mhat64"]).max() <= 256
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 2.0 ** -4, 1.0, "bf16")
    np.testing.assert_array_equal(got["Mhat"], ref["Mhat64"].astype(np.float32))
    cfg = synth.CONFIGS["tiny"].with_(G=G)
    J = [synth.ids_for(cfg, g) for g in range(G)]
    Dl = [synth.grad_values(cfg.K, cfg.D, "signed", rank=g).numpy() for g in range(G)]
    E0 = synth.table_values(cfg.V, cfg.D, "signed").numpy()
    ref = oracle.sync_unique(J, Dl, E0.copy(), 0.1)
    got = oracle.sync_unique_compressed(J, Dl, E0.copy(), 0.1, 1.0, "bf16")
    absM = sum(np.abs(m) for m in ref["M"])
    bound = 2.0 ** -7 * (absM + np.abs(ref["Mhat64"])) + 1e-37
    assert (np.abs(got["Mhat"].astype(np.float64) - ref["Mhat64"]) <= bound).all()
