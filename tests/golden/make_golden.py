"""Generate tests/golden/golden.json — TEST INFRASTRUCTURE.

The reference (C++/Eigen/FFTW) cannot be built or imported in this image
(SURVEY §8(c)), so these fixtures come from a second, independent
restatement written here in plain Python/numpy (no shared code with the C++
oracle): pure-Python std::mt19937_64 and libstdc++'s polar-method
normal_distribution (reference rng.hpp:12-38), the quintic weights evaluated
from the piecewise formulas of interpolation.cpp:15-39 with numpy.polyval,
Grid::cover (interpolation.cpp:117-146), and a dense D-SKI matrix
B·K_UU·Bᵀ + noise assembled with numpy (test_dski.cpp:34-47). The C++ oracle
must reproduce every case to 1e-13 (tests/test_oracle_pins.py).

Run:  python tests/golden/make_golden.py
"""
import json
import math
import os

import numpy as np

M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 ([rand.predef]): w=64 n=312 m=156 r=31."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & M64
        self.idx = 312

    def __call__(self):
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


def mix_seed(seed, stream):
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rademacher(n, seed, stream):
    g = MT19937_64(mix_seed(seed, stream))
    return [1.0 if (g() & 1) else -1.0 for _ in range(n)]


def canonical(g):
    # libstdc++ generate_canonical<double,53> over a 64-bit engine: one draw,
    # r / 2^64 rounded to double, clamped below 1.
    r = g()
    v = float(r) / 18446744073709551616.0
    if v >= 1.0:
        v = math.nextafter(1.0, 0.0)
    return v


def gaussian(n, seed, stream):
    """libstdc++ normal_distribution (Marsaglia polar; returns y*mult first,
    caches x*mult)."""
    g = MT19937_64(mix_seed(seed, stream))
    out, saved = [], None
    while len(out) < n:
        if saved is not None:
            out.append(saved)
            saved = None
            continue
        while True:
            x = 2.0 * canonical(g) - 1.0
            y = 2.0 * canonical(g) - 1.0
            r2 = x * x + y * y
            if r2 <= 1.0 and r2 != 0.0:
                break
        mult = math.sqrt(-2.0 * math.log(r2) / r2)
        saved = x * mult
        out.append(y * mult)
    return out


P1 = np.array([-25.0, 63.0, -35.0, -15.0, 0.0, 12.0]) / 12.0  # on [0,1)
P2 = np.polymul(np.polymul([1.0, -2.0], [1.0, -1.0]), [25.0, -114.0, 153.0, -48.0]) / 24.0
P3 = -np.polymul(np.polymul(np.polymul([1.0, -3.0], [1.0, -3.0]), [1.0, -3.0]),
                 np.polymul([1.0, -2.0], [5.0, -8.0])) / 24.0


def qpiece(s):
    s = abs(s)
    if s < 1:
        return np.polyval(P1, s)
    if s < 2:
        return np.polyval(P2, s)
    if s < 3:
        return np.polyval(P3, s)
    return 0.0


def qderiv(s):
    sg = -1.0 if s < 0 else 1.0
    a = abs(s)
    if a < 1:
        v = np.polyval(np.polyder(P1), a)
    elif a < 2:
        v = np.polyval(np.polyder(P2), a)
    elif a < 3:
        v = np.polyval(np.polyder(P3), a)
    else:
        v = 0.0
    return sg * v


def quintic(t):
    args = [t - (k - 2) for k in range(6)]
    return [qpiece(a) for a in args], [qderiv(a) for a in args]


def cover(X, target, margin, max_nodes):
    n, d = X.shape
    dims, origin, spacing = [], [], []
    for j in range(d):
        lo, hi = X[:, j].min(), X[:, j].max()
        span = max(hi - lo, 1e-12)
        h = target
        m = int(math.ceil(span / h)) + 1 + 2 * margin
        if m > max_nodes:
            m = max_nodes
            h = span / (m - 1 - 2 * margin)
        m = max(m, 6 + 2 * margin)
        dims.append(m)
        spacing.append(h)
        origin.append(lo - margin * h)
    return dims, np.array(origin), np.array(spacing)


def dense_dski(X, ell, s, noise, dims, origin, spacing):
    n, d = X.shape
    M = int(np.prod(dims))
    B = np.zeros((n * (d + 1), M))
    for i in range(n):
        axes = []
        for j in range(d):
            sv = (X[i, j] - origin[j]) / spacing[j]
            cell = math.floor(sv)
            w, dw = quintic(sv - cell)
            axes.append((cell - 2, np.array(w), np.array(dw) / spacing[j]))
        for c in np.ndindex(*([6] * d)):
            flat = 0
            for j in range(d):
                flat = flat * dims[j] + axes[j][0] + c[j]
            B[i, flat] = np.prod([axes[j][1][c[j]] for j in range(d)])
            for p in range(d):
                B[(p + 1) * n + i, flat] = np.prod(
                    [axes[j][2][c[j]] if j == p else axes[j][1][c[j]] for j in range(d)])
    P = np.array([origin + np.array(ix) * spacing for ix in np.ndindex(*dims)])
    D2 = ((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)
    K = s * s * np.exp(-0.5 * D2 / ell ** 2)
    nd = np.r_[np.full(n, noise[0] ** 2), np.full(n * d, noise[1] ** 2)]
    return B @ K @ B.T + np.diag(nd)


def main():
    cases = []
    for t in (0.0, 0.25, 0.5, 0.8125):
        w, dw = quintic(t)
        cases.append({"name": f"quintic_{t}", "kind": "quintic", "t": t, "out": list(w) + list(dw),
                      "tol": 1e-13})
    for seed, stream in ((0, 0), (0, 1000), (7, 50003)):
        cases.append({"name": f"rademacher_{seed}_{stream}", "kind": "rademacher", "n": 64,
                      "seed": seed, "stream": stream, "out": rademacher(64, seed, stream), "tol": 0.0})
        cases.append({"name": f"gaussian_{seed}_{stream}", "kind": "gaussian", "n": 64,
                      "seed": seed, "stream": stream, "out": gaussian(64, seed, stream), "tol": 0.0})
    rng = np.random.default_rng(2024)
    for n, d, ell, s, noise, spacing, maxn in ((25, 2, 0.5, 1.1, (0.1, 0.05), 0.125, 14),
                                               (12, 1, 0.4, 1.3, (0.2, 0.3), 0.05, 30)):
        X = rng.uniform(0, 1, (n, d))
        dims, origin, h = cover(X, spacing, 3, maxn)
        A = dense_dski(X, ell, s, noise, dims, origin, h)
        v = rng.standard_normal(A.shape[0])
        cases.append({"name": f"dski_mvm_d{d}", "kind": "dski_mvm", "X": X.tolist(), "ell": ell,
                      "s": s, "noise": list(noise), "spacing": spacing, "max_nodes": maxn,
                      "v": v.tolist(), "out": (A @ v).tolist(),
                      # expanded-polynomial weights round differently from the
                      # reference's nested forms: agreement is to ~1e-13
                      "tol": 2e-12})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "cases": cases}, f)
    print(f"wrote {len(cases)} cases to {path}")


if __name__ == "__main__":
    main()
