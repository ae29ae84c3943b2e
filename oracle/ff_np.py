"""TEST INFRASTRUCTURE ONLY — finite-field arithmetic GF(p), p = 2^31 - 1, in numpy.

Bit-identical to the device number system `NFF` in
paper_2604_15272_b200/csrc/sgm_dev.cuh:
  add / mul / square       exact modular arithmetic
  div(a, b)                a * b^(p-2)   (so div by 0 gives 0; same on device)
  scale(x, n/d)            x * (n * d^(p-2))
  exp / silu / sqrt        uninterpreted keyed hashes h_k(x) = mix64(x + K_k) mod p
  sum / matmul             exact sums mod p
Why this is a sound equivalence check: every rewrite rule the reference's
verifier uses (symfuse verifier/axioms.py:75-355) holds in any field with
uninterpreted unary functions; no rule relies on exp/silu/sqrt identities.
"""
from __future__ import annotations

import numpy as np

P = (1 << 31) - 1
_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
KEY = {"exp": 0x9E3779B97F4A7C15, "silu": 0x3C6EF372FE94F82A, "sqrt": 0xDAA66D2C7DDF743F}


def mix64(z):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def mix64_int(z: int) -> int:
    z &= _M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    z ^= z >> 31
    return z


def ff_uniform(n: int, seed: int, salt: int) -> np.ndarray:
    """value(i) = mix64(key + i*GOLDEN) mod p, key = mix64(seed ^ mix64(salt));
    the device twin is sgm_ff_fill (include/sgm.h)."""
    key = mix64_int((seed & _M64) ^ mix64_int(salt))
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = mix64(np.uint64(key) + i * np.uint64(GOLDEN))
    return (v % np.uint64(P)).astype(np.int64)


def reduce(x) -> np.ndarray:
    return np.asarray(x, dtype=np.int64) % P


def inv(x):
    """x^(p-2) mod p, vectorised square-and-multiply (int64 products < 2^62)."""
    x = reduce(x)
    r = np.ones_like(x)
    b = x.copy()
    e = P - 2
    while e:
        if e & 1:
            r = (r * b) % P
        b = (b * b) % P
        e >>= 1
    return r


def const(num: int, den: int) -> int:
    return (num % P) * pow(den % P, P - 2, P) % P


def hash_op(kind: str, x) -> np.ndarray:
    with np.errstate(over="ignore"):
        v = mix64(reduce(x).astype(np.uint64) + np.uint64(KEY[kind]))
    return (v % np.uint64(P)).astype(np.int64)


def matmul(a, b) -> np.ndarray:
    """Exact (a @ b) mod p.  Both operands are split into 11-bit limbs and the
    9 limb products run as float64 BLAS GEMMs: every partial sum is an integer
    below K * 2^22 < 2^53 (K < 2^31), so the float result is exact."""
    a, b = reduce(a), reduce(b)
    out = np.zeros(np.broadcast_shapes(a.shape[:-2], b.shape[:-2]) + (a.shape[-2], b.shape[-1]), dtype=np.int64)
    al = [((a >> s) & 0x7FF).astype(np.float64) for s in (0, 11, 22)]
    bl = [((b >> s) & 0x7FF).astype(np.float64) for s in (0, 11, 22)]
    for i in range(3):
        for j in range(3):
            part = np.matmul(al[i], bl[j]).astype(np.int64) % P
            out = (out + part * pow(2, 11 * (i + j), P)) % P
    return out


class FFArith:
    """Op table with the same signature as symfuse interp.apply_op (interp.py:45-66)."""

    name = "ff"

    def __call__(self, kind, args, axis=None, const_=None):
        if kind in ("exp", "silu", "sqrt"):
            return hash_op(kind, args[0])
        if kind == "square":
            a = reduce(args[0])
            return (a * a) % P
        if kind == "scale":
            return (reduce(args[0]) * const(const_.numerator, const_.denominator)) % P
        if kind == "sum":
            return reduce(args[0]).sum(axis=axis, keepdims=True) % P
        if kind == "matmul":
            return matmul(args[0], args[1])
        if kind == "div":
            return (reduce(args[0]) * inv(args[1])) % P
        if kind == "mul":
            return (reduce(args[0]) * reduce(args[1])) % P
        if kind == "add":
            return (reduce(args[0]) + reduce(args[1])) % P
        raise ValueError(f"unknown op kind {kind}")

    def accum(self, acc, val):
        return (reduce(acc) + reduce(val)) % P

    def zeros(self, like):
        return np.zeros(np.shape(like), dtype=np.int64)

    def cast(self, arr):
        return reduce(arr)

    def fill(self, dims):
        return np.full(dims, -1, dtype=np.int64)  # not a residue: unwritten cells never match
