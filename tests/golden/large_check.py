"""Size-independent parity checks for the configs too large to store the reference output
(cfg3: N = 6,291,456; cfg4: the spheroid). TEST / CHECK INFRASTRUCTURE ONLY.

A fixture (`tests/golden/<cfg>_large.npz`, written by `make_large.py` from the reference
itself) stores, for the reference's S and D without the RP term (layer_potentials minus
rp_singular_apply, solver.cpp:78-147):

* K = 64 random projections  p_k = sum_t w_kt S_t  over ALL N targets, with weights
  w_kt = (+-1 +- i)/sqrt(2) drawn from a counter-based hash (splitmix64 of k, t), so the
  GPU side regenerates them without storing them. For a difference vector e = S_gpu - S_ref,
  E|w_k . e|^2 = ||e||^2, so  sqrt(mean_k |p_k(gpu) - p_k(ref)|^2) / ||S_ref||  estimates the
  full-vector relative L2 error (relative spread ~ 1/sqrt(2K) ~ 9%);
* S and D exactly at 65,536 seeded sample targets (max-abs and sample rel-L2);
* the RP term at a sub-sample of targets, from the reference's own beta_precompute and
  rp_singular_apply over those targets' pairs (independent of the GPU beta tables);
* plan fingerprints: per-level relevant-segment hashes and counts, the Morton permutation
  hash, the pair count, and the product CPU planner's per-level decision hashes.
"""
from __future__ import annotations

import numpy as np

K_PROJ = 64
SAMPLE = 65536
RP_SAMPLE = 16384
_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def seq_hash(v) -> int:
    """sum_i splitmix64(v_i + splitmix64(i)) mod 2^64 (oracle/ref_driver.cpp ref_plan_*_hash)"""
    v = np.asarray(v).astype(np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum(_splitmix64(v + _splitmix64(np.arange(len(v), dtype=np.uint64))), dtype=np.uint64))


def segment_hash(seg_box, seg_gamma) -> int:
    b = np.asarray(seg_box).astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    g = np.asarray(seg_gamma).astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    return seq_hash((b << np.uint64(32)) | g)


def weights(k: int, t0: int, t1: int) -> np.ndarray:
    """w_kt for t in [t0, t1): (+-1 +- i)/sqrt(2), sign bits from splitmix64((k << 40) + t)"""
    t = np.arange(t0, t1, dtype=np.uint64) + (np.uint64(k) << np.uint64(40))
    h = _splitmix64(t)
    re = 1.0 - 2.0 * ((h >> np.uint64(17)) & np.uint64(1)).astype(np.float64)
    im = 1.0 - 2.0 * ((h >> np.uint64(43)) & np.uint64(1)).astype(np.float64)
    return (re + 1j * im) * np.sqrt(0.5)


def projections(v: np.ndarray, k_proj: int = K_PROJ, chunk: int = 1 << 21) -> np.ndarray:
    n = len(v)
    out = np.zeros(k_proj, dtype=np.complex128)
    for k in range(k_proj):
        acc = 0j
        for t0 in range(0, n, chunk):
            t1 = min(n, t0 + chunk)
            acc += np.dot(weights(k, t0, t1), v[t0:t1])
        out[k] = acc
    return out


def sample_targets(n: int, count: int = SAMPLE, seed: int = 20112) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.unique(rng.choice(n, size=min(count, n), replace=False)).astype(np.int64)


def rp_sample_targets(sample: np.ndarray, count: int = RP_SAMPLE) -> np.ndarray:
    return sample[:: max(1, len(sample) // count)][:count]


def compare(fix, S: np.ndarray, D: np.ndarray) -> dict:
    """S, D: the GPU's layer potentials WITHOUT the RP term (original order, full length)."""
    res = {}
    idx = fix["sample_idx"]
    for name, v in (("S", S), ("D", D)):
        p = projections(v, len(fix[f"proj{name}"]))
        err = np.sqrt(np.mean(np.abs(p - fix[f"proj{name}"]) ** 2))
        ref_s = fix[f"{name}_sample"]
        d = v[idx] - ref_s
        res[name] = {
            "rel_l2_est_full": float(err / fix[f"norm{name}"]),
            "rel_l2_sample": float(np.linalg.norm(d) / np.linalg.norm(ref_s)),
            "max_abs_sample": float(np.max(np.abs(d))),
            "rel_norm_diff": float(abs(np.linalg.norm(v) - fix[f"norm{name}"]) / fix[f"norm{name}"]),
        }
    return res


def compare_rp(fix, rpS: np.ndarray, rpD: np.ndarray) -> dict:
    """rpS, rpD: the GPU's RP term at fix['rp_idx'] (original order)"""
    out = {}
    for name, v in (("S", rpS), ("D", rpD)):
        ref = fix[f"rp{name}"]
        out[name] = {"rel_l2_sample": float(np.linalg.norm(v - ref) / np.linalg.norm(ref)),
                     "max_abs_sample": float(np.max(np.abs(v - ref)))}
    return out
