"""Write tests/golden/lattice_moments.txt: exact Chebyshev moments of the infinite
periodic nearest-neighbour lattice (the paper's model) in 1D/2D/3D.

Independent of oracle/ and of the CUDA path: pure integer combinatorics in exact
rational arithmetic.

* <i|H^k|i> for hopping t counts closed walks of length k from a site, times t^k.
  Closed walks of length 2k: 1D  C(2k,k); 2D  C(2k,k)^2;
  3D  sum_{i+j+l=k} (2k)! / (i!^2 j!^2 l!^2); odd lengths: 0 (bipartite).
* H~ = H / a with a = 2 * ndim |t| (Gerschgorin, Eq 8-9 with b = 0).
* T_n(x) = sum_k c_{n,k} x^k from T_0 = 1, T_1 = x, T_{n+2} = 2x T_{n+1} - T_n
  (Eq 4-5), so mu_n = (1/D) Tr T_n(H~) = sum_k c_{n,k} <H~^k>  (Eq 13).
For a finite periodic lattice with every extent L > n a closed walk of length n
cannot wind around the torus, so the finite-L moments equal these for n < L.
"""
from fractions import Fraction
from math import comb, factorial
import os

NMAX = 48


def closed_walks(ndim: int, k: int) -> int:
    if k % 2:
        return 0
    h = k // 2
    if ndim == 1:
        return comb(2 * h, h)
    if ndim == 2:
        return comb(2 * h, h) ** 2
    total = 0
    for i in range(h + 1):
        for j in range(h + 1 - i):
            l = h - i - j
            total += factorial(2 * h) // (factorial(i) ** 2 * factorial(j) ** 2 * factorial(l) ** 2)
    return total


def cheb_coeffs(nmax: int):
    T = [[1], [0, 1]]
    for n in range(2, nmax + 1):
        prev, cur = T[n - 2], T[n - 1]
        nxt = [0] * (n + 1)
        for k, c in enumerate(cur):
            nxt[k + 1] += 2 * c
        for k, c in enumerate(prev):
            nxt[k] -= c
        T.append(nxt)
    return T


def moments(ndim: int, nmax: int):
    a = 2 * ndim
    T = cheb_coeffs(nmax)
    out = []
    for n in range(nmax + 1):
        s = Fraction(0)
        for k, c in enumerate(T[n]):
            if c:
                s += c * Fraction(closed_walks(ndim, k), a ** k)  # t^k = 1 for even k
        out.append(s)
    return out


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "lattice_moments.txt"), "w") as f:
        f.write("# ndim n mu_n  -- exact Chebyshev moments of the infinite periodic\n")
        f.write("# nearest-neighbour lattice, a = 2*ndim|t|, b = 0 (Eq 13, PAPER.md:99-105;\n")
        f.write("# model PAPER.md:229).  Written by make_lattice_moments.py (combinatorics only).\n")
        for ndim in (1, 2, 3):
            for n, m in enumerate(moments(ndim, NMAX)):
                f.write(f"{ndim} {n} {float(m)!r}\n")
