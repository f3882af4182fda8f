"""Fit the element-math polynomials of plg_math.cuh (near-minimax, mpmath Chebyshev fits),
round them to doubles and report their maximum errors on the reduced ranges.

    python tools/fit_polys.py

exp(-2r), |r| <= ln2/512 ; exp(-r/2), |r| <= ln2/128 ; log1p(r)/r, |r| <= 1/(2*256+1).
"""

import mpmath as mp

mp.mp.dps = 50


def fit(f, lo, hi, deg):
    coeffs, err = mp.chebyfit(f, [lo, hi], deg + 1, error=True)
    coeffs = [float(c) for c in coeffs]  # highest degree first
    # error of the double-rounded polynomial, sampled densely, in high precision
    worst = mp.mpf(0)
    N = 4000
    for i in range(N + 1):
        x = lo + (hi - lo) * i / N
        p = mp.mpf(0)
        for c in coeffs:
            p = p * x + mp.mpf(c)
        worst = max(worst, abs(p - f(x)) / abs(f(x)))
    return coeffs, float(worst)


def main():
    ln2 = mp.log(2)
    specs = [
        ("exp(-2r)", lambda r: mp.exp(-2 * r), -ln2 / 512, ln2 / 512),
        ("exp(-r/2)", lambda r: mp.exp(-r / 2), -ln2 / 128, ln2 / 128),
        ("log1p(r)/r", lambda r: mp.log1p(r) / r if r != 0 else mp.mpf(1), -mp.mpf(1) / 513, mp.mpf(1) / 513),
    ]
    for name, f, lo, hi in specs:
        for deg in (3, 4, 5):
            coeffs, err = fit(f, lo, hi, deg)
            print(f"{name:12s} deg {deg}: max rel err {err:.3e}  coeffs (high->low) {coeffs}")


if __name__ == "__main__":
    main()


def short(x):
    """Round to a double whose low 32 bits are zero (a DMUL/DADD 32-bit immediate)."""
    import struct

    bits = struct.unpack("<Q", struct.pack("<d", float(x)))[0]
    lo = bits & 0xFFFFFFFF
    bits = (bits >> 32) << 32
    if lo >= 0x80000000:
        bits += 1 << 32
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def fit_short_lead(f, lo, hi, deg):
    """Near-minimax fit whose leading coefficient is a short double (immediate operand):
    fit deg first, round the leading coefficient, refit the rest to f - c x^deg."""
    coeffs, _ = fit(f, lo, hi, deg)
    c = short(coeffs[0])
    rest, _ = fit(lambda x: f(x) - mp.mpf(c) * x ** deg, lo, hi, deg - 1)
    full = [c] + rest
    worst = mp.mpf(0)
    N = 4000
    for i in range(N + 1):
        x = lo + (hi - lo) * i / N
        p = mp.mpf(0)
        for cc in full:
            p = p * x + mp.mpf(cc)
        worst = max(worst, abs(p - f(x)) / abs(f(x)))
    return full, float(worst)
