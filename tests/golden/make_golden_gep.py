"""Golden fixtures for MTNUFFT0 from the REFERENCE (O(N^3): small N only).

  gep_gpss.npz  gpss_exact (tapers.cpp:118-144) on jittered grids (the reference's own
                generate_grid) at N = 256, 512, 1024, real nominal band (f_c = 0), K = 7,
                plus N = 256 with a complex band (f_c != 0); weights [K][N] complex + concentrations
  gep_pencil.npz generalized_hermitian_eigen (eig.cpp:612-659) on a random Hermitian A and
                an SPD M (N = 128): values, vectors, residuals
  gep_mtnufft0.npz MtnufftEstimator(taper_mode = exact_nominal) P(f) at N = 1024 (estimators.cpp:91-122)

Run in the build container: python tests/golden/make_golden_gep.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import REF, build  # noqa: E402


def main():
    build(ref=True)
    out = {}
    for n in (256, 512, 1024):
        t = REF.generate_grid(1, n, seed=100 + n)
        span = t[-1] - t[0]
        f_max = 0.5 * n / span
        f_w = 4.0 / span
        w, conc = REF.gpss_exact(t, f_max, 0.0, f_w, 7)
        out.update({f"t{n}": t, f"fmax{n}": f_max, f"fw{n}": f_w, f"w{n}": w, f"conc{n}": conc})
    t = REF.generate_grid(1, 256, seed=77)
    span = t[-1] - t[0]
    f_max, f_w, f_c = 0.5 * 256 / span, 3.0 / span, 0.2 * 256 / span
    w, conc = REF.gpss_exact(t, f_max, f_c, f_w, 5)
    out.update({"tc": t, "fmaxc": f_max, "fwc": f_w, "fcc": f_c, "wc": w, "concc": conc})
    np.savez_compressed(os.path.join(HERE, "gep_gpss.npz"), **out)

    rng = np.random.default_rng(11)
    n = 128
    b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (b + b.conj().T) / 2
    a = a / np.abs(np.linalg.eigvalsh(a)).max() * 0.45 + 0.5 * np.eye(n)  # spectrum inside [0, 1]
    c = rng.standard_normal((n, n))
    m = c @ c.T / n + np.eye(n)
    vals, vecs, res = REF.generalized_eigen(a, m, 6)
    np.savez_compressed(os.path.join(HERE, "gep_pencil.npz"), a=a, m=m, values=vals, vectors=vecs, residuals=res)

    n = 1024
    t = REF.generate_grid(1, n, seed=5)
    span = t[-1] - t[0]
    f_max = 0.5 * n / span
    f_w = 4.0 / span
    x = REF.rng_gauss(99, n)
    centers = np.arange(256) * (f_max / 256)
    p, w, method = REF.mtnufft0(t, x, f_max, centers, f_w, 7, 1e-9)
    np.savez_compressed(os.path.join(HERE, "gep_mtnufft0.npz"), t=t, x=x, f_max=f_max, f_w=f_w, centers=centers,
                        power=p, tapers=w, method=method)
    print("wrote gep_gpss.npz gep_pencil.npz gep_mtnufft0.npz")


if __name__ == "__main__":
    main()
