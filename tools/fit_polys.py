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
