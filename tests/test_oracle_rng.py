"""Pins of the oracle's RNG layer (contract readings R1, R2, R4)."""
import math
import os
import subprocess
import tempfile

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(O):
    for ctr, key, want in _kat():
        assert O.philox4x32_10(ctr, key).tolist() == want


CURAND_HOST = r"""
#include <cstdio>
#include <cstdlib>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main(int argc, char** argv) {
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < 2000; i++) {
    unsigned w[6];
    for (int k = 0; k < 6; k++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; w[k] = (unsigned)(s >> 11); }
    uint4 c = {w[0], w[1], w[2], w[3]}; uint2 key = {w[4], w[5]};
    uint4 o = curand_Philox4x32_10(c, key);
    printf("%u %u %u %u %u %u %u %u %u %u\n", w[0], w[1], w[2], w[3], w[4], w[5], o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""


def test_philox_matches_curand_host_build(O):
    """Independent implementation: cuRAND's curand_Philox4x32_10 (curand_philox4x32_x.h:171),
    compiled for the HOST with g++ (test-only use of the header)."""
    inc = "/usr/local/cuda/include"
    if not os.path.exists(os.path.join(inc, "curand_philox4x32_x.h")):
        pytest.skip("cuRAND headers not present")
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "k.cpp"), os.path.join(d, "k")
        open(src, "w").write(CURAND_HOST)
        r = subprocess.run(["g++", "-O1", "-I", inc, src, "-o", exe], capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("cannot host-compile curand header: " + r.stderr[-300:])
        out = subprocess.check_output([exe], text=True)
    n = 0
    for line in out.splitlines():
        v = [int(t) for t in line.split()]
        assert O.philox4x32_10(v[:4], v[4:6]).tolist() == v[6:10]
        n += 1
    assert n == 2000


def test_u01_exact_endpoints(O):
    # u01(k) = (k + 0.5) 2^-32: exact, strictly inside (0, 1)   (reading R2)
    assert O.u01(0) == 2.0 ** -33
    assert O.u01(2**32 - 1) == 1.0 - 2.0 ** -33
    assert O.u01(2**31) == 0.5 + 2.0 ** -33
    ks = np.random.default_rng(0).integers(0, 2**32, 1000)
    vals = [O.u01(int(k)) for k in sorted(ks)]
    assert all(0 < a <= b < 1 for a, b in zip(vals, vals[1:]))


def _count_skip_ge(O, h, ell):
    """#{k in [0, 2^32): skip(k, h) >= ell}, using that skip is non-increasing in k."""
    lo, hi = 0, 2**32  # predicate true on [0, K)
    while lo < hi:
        mid = (lo + hi) // 2
        s = O.skip(mid, h)
        if s == -1 or s >= ell:
            lo = mid + 1
        else:
            hi = mid
    return lo


@pytest.mark.parametrize("q", [1e-6, 0.01, 0.3, 0.9, 0.999999])
def test_skip_law_exact_enumeration(O, q):
    """P(L >= ell) over ALL 2^32 words equals (1-q)^ell (Fig. 2 caption), up to
    the 2^-32 resolution of u01: the geometric law of the skip is exact, not approximate."""
    h = -math.log1p(-q)
    # monotonicity of the predicate on a random subset (needed by the counting search)
    ks = np.sort(np.random.default_rng(1).integers(0, 2**32, 4000))
    sk = [O.skip(int(k), h) for k in ks]
    sk = [s if s >= 0 else 2**62 for s in sk]
    assert all(a >= b for a, b in zip(sk, sk[1:]))
    ells = sorted(set([0, 1, 2, 3, 5, 10, 20, 50] + [int(m / q) for m in (0.1, 0.5, 1, 2, 5)]))
    for ell in ells:
        P = _count_skip_ge(O, h, ell) / 2.0**32
        want = math.exp(-ell * h)  # (1-q)^ell
        if want < 2.0 ** -32 * 4:
            continue  # below word resolution (tail truncated at E <= 22.9, reading R2)
        assert abs(P - want) <= 2.0 ** -32 + 1e-12 * want, (q, ell, P, want)


def test_skip_special_values(O):
    # q = 1 (h = inf): every skip is 0 -> L = 1 always ("q = 1 -> always 1")
    for k in (0, 1, 2**31, 2**32 - 1):
        assert O.skip(k, math.inf) == 0
    # q = 0 (h = 0): R = +inf -> no candidate is ever reached (reading R5)
    assert O.skip(12345, 0.0) == -1
