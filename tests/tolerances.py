"""Float-parity metric.

north_star: "within max relative error 1e-5 (fp32 accumulation)".  Made
well-defined per value mode:

* INT    -- every partial sum is an exact fp32 integer: bit-exact.
* POS    -- all terms positive (condition number 1): |g - r| <= 1e-5 |r|.
* SIGNED -- terms cancel; relative error against |r| is ill-posed, so the
            bound is the standard summation-error scale:
            |g - r| <= 1e-5 * A, A = sum |contributions| (fp64, oracle side).
For updated table rows the scale is |E0| + lr * A.
"""
import numpy as np

RTOL = 1e-5


def check_rows(got, ref64, absscale64, mode, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref64, np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if mode == "int":
        bad = np.argwhere(got != ref)
        assert bad.size == 0, f"{what}: {len(bad)} non-bit-exact, first {bad[:3].tolist()}"
        return 0.0
    err = np.abs(got - ref)
    if mode == "pos":
        scale = np.abs(ref)
    else:
        scale = np.asarray(absscale64, np.float64)
    scale = np.maximum(scale, np.finfo(np.float32).tiny)
    rel = err / scale
    worst = float(rel.max()) if rel.size else 0.0
    assert worst <= RTOL, f"{what}: max scaled error {worst:.3e} > {RTOL}"
    return worst


def compressed_tol(absscale64, F, G):
    """Bound on |GPU - oracle| for a row of M^ from the compressed exchange
    (R15 / "Tolerances"): each side is within
    2^-10 (sum_g |M_g| + |M^|) + (G + 1) 2^-24 / F of the exact sum (one
    binary16 rounding per transfer, pinned in tests/test_compression_oracle.py),
    and sum_g |M_g|, |M^| <= A, so the two sides differ by at most
    2^-8 A + (G + 1) 2^-23 / F."""
    return 2.0 ** -8 * np.asarray(absscale64, np.float64) + (G + 1) * 2.0 ** -23 / F


def check_compressed_rows(got, ref, tol, what="", min_exact=0.99):
    """|got - ref| <= tol everywhere, and at least `min_exact` of the elements
    bit-identical (the two sides differ only where an fp32 summation-order
    difference crosses a binary16 rounding boundary)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    assert (err <= tol).all(), f"{what}: max err {err.max():.3e}, tol at worst {tol.ravel()[np.argmax(err - tol)]:.3e}"
    if got.size:
        frac = float((got == ref).mean())
        assert frac >= min_exact, f"{what}: only {frac:.4f} of elements bit-identical"
