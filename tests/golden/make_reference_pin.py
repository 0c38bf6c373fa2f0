"""Generates tests/golden/reference_pin.json: the reference's own outputs
(oracle/_ref — the reference headers compiled unchanged against the
Eigen-API shim) and the CAS oracle's bit-level digests at the five
BASELINE.json config shapes, on the seed-0 trial-0 start frame of each config,
at delta values of the config's default schedule.

TEST INFRASTRUCTURE.  Run here (where /root/reference exists):
    python tests/golden/make_reference_pin.py
The JSON travels with the repo; the GPU tests compare the CUDA path against
it (tests/test_gpu_reference_pin.py) without needing the reference on the box.

Stored per (config, delta):
  * frame_sha256: sha256 of the start frame bytes (random_frame of
    SplitMix64(mix_seed(0, 0)); real configs draw normal() per entry), so the
    consumer can check its RNG reproduces the same input;
  * ref: F, s, |grad|, 128 gradient entries at seeded positions, 4
    projections grad . r_j (r_j ~ N(0,1), numpy default_rng(1000 + j)),
    coherence mu of the frame and its first-argmax pair;
  * cas: sha256 of the CAS oracle's F, s and gradient bits (the bit-level
    contract the GPU must meet) and the CAS F, s;
  * hvp (configs 1-4, direction r_0 / 256 — an exact scaling, so every
    platform forms the same input bits): reference
    |Hv| and 128 samples, CAS sha256.
"""
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2207_06374_b200 import abi  # noqa: E402
from tests import oracle_ffi as O  # noqa: E402
from tests import ref_ffi as R  # noqa: E402

CONFIGS = {"c1": (abi.REAL, 4, 10), "c2": (abi.COMPLEX, 2, 100), "c3": (abi.COMPLEX, 6, 36),
           "c4": (abi.REAL, 64, 1024), "c5": (abi.COMPLEX, 128, 4096)}
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_pin.json")
NSAMP = 128


def lanes(field, d, N):
    """trstmi_lanes() of the product for these shapes, stated
    here so the generator does not load the product library."""
    return {(1, 4, 10): 64, (0, 2, 100): 512, (0, 6, 36): 128, (1, 64, 1024): 32768,
            (0, 128, 4096): 32768}[(field, d, N)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def probes(dim):
    idx = np.sort(np.random.default_rng(7).choice(dim, size=min(NSAMP, dim), replace=False))
    rs = [np.random.default_rng(1000 + j).standard_normal(dim) for j in range(4)]
    return idx, rs


def schedule_points(N):
    s = R.schedule(N)
    return sorted({s[0], s[len(s) // 2], s[-1]}, reverse=True)


def main(only=None):
    out = {"generator": "tests/golden/make_reference_pin.py", "nsamp": NSAMP, "configs": {}}
    if os.path.exists(OUT):
        out = json.load(open(OUT))
    for name, (field, d, N) in CONFIGS.items():
        if only and name not in only:
            continue
        dim = abi.dim_of(field, d, N)
        x = O.random_frames(field, d, N, 0, 0, 1)[0][0]
        if field == abi.COMPLEX:  # the reference's own random_frame must produce the same start frame
            cfg = abi.default_cfg(field, d, N)
            b = R.Batch(cfg, 0, 0, 1)
            xr, _ = b.params()
            b.close()
            # same Box-Muller draws; the column norms differ only in summation order (the shim's
            # sequential sum vs the CAS fma chain), i.e. by at most an ulp of each entry
            assert np.max(np.abs(xr[0] - x)) <= 4.5e-16, "reference random_frame differs from the restated RNG"
        idx, rs = probes(dim)
        mu, arg, zc = R.coherence(field, d, N, x, normalize=False)
        entry = {"field": field, "d": d, "N": N, "seed": 0, "trial": 0, "frame_sha256": sha(x),
                 "sample_idx": idx.tolist(),
                 "ref_random_frame_max_abs_diff": float(np.max(np.abs(xr[0] - x))) if field == abi.COMPLEX else None,
                 "mu": mu, "argmax_pair": arg, "evals": []}
        S = lanes(field, d, N)
        for delta in schedule_points(N):
            t0 = time.time()
            F, s, g, _, z = R.eval_objective(field, d, N, x, delta)
            Fo, so, go, _, zo = O.eval_objective(field, d, N, S, x, delta)
            assert z == -1 and zo == -1
            e = {"delta": delta,
                 "ref": {"F": F, "s": s, "gnorm": float(np.linalg.norm(g)), "g_samples": g[idx].tolist(),
                         "proj": [float(np.dot(g, r)) for r in rs]},
                 "cas": {"F": Fo, "s": so, "F_bits_sha256": sha([Fo, so]), "grad_sha256": sha(go)}}
            rel = abs(F - Fo) / abs(F)
            grel = np.linalg.norm(g - go) / np.linalg.norm(g)
            e["cas_vs_ref"] = {"F_rel": rel, "grad_rel_l2": float(grel),
                               "grad_componentwise": float(np.max(np.abs(g - go) / np.maximum(np.abs(g), 1.0)))}
            if N <= 1024:
                v = rs[0] * 0.00390625  # exact power-of-two scaling: no platform-dependent norm in the input
                hv, hz = R.hvp(field, d, N, x, v, delta)
                ho, path, hoz = O.hvp(field, d, N, S, x, v, delta)
                e["hvp"] = {"ref_norm": float(np.linalg.norm(hv)), "ref_samples": hv[idx].tolist(),
                            "cas_sha256": sha(ho),
                            "cas_vs_ref_rel_l2": float(np.linalg.norm(hv - ho) / np.linalg.norm(hv))}
            entry["evals"].append(e)
            print(name, "delta=%.3g" % delta, "F_rel=%.2e grad_rel=%.2e" % (rel, grel), "%.1fs" % (time.time() - t0),
                  flush=True)
        out["configs"][name] = entry
        json.dump(out, open(OUT, "w"), indent=1)
    return out


if __name__ == "__main__":
    main(sys.argv[1:] or None)
