"""Oracle side of the full-size parity tests (tests/test_gpu_fullsize.py):
runs oracle.solve on a BASELINE config at full size and writes what the GPU
result is compared with -- the Fiedler vector, lambda_2, the residual, and a
SHA-256 digest of every level's hierarchy arrays (CSR pattern and values,
matching, aggregate ids, colours).  Calls only graphgen/ and oracle/.

    python tests/oracle_fullsize.py CONFIG OUT_PREFIX

writes OUT_PREFIX.json and OUT_PREFIX.vec.npy.  Config 4 (8192^2 grid) takes
~6 min and ~14 GB of host memory, config 3 (256^3 grid) ~2.5 min and ~5 GB.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# canonical dtypes of the digested arrays (both sides convert before hashing)
DTYPES = {"rp": np.int64, "ci": np.int32, "w": np.float64, "agg": np.int64, "mate": np.int64,
          "color": np.int32}


def digest(a, key):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=DTYPES[key]).tobytes()).hexdigest()


def level_digests(rp, ci, w, color, agg=None, mate=None):
    d = {"n": int(rp.size - 1), "nnz": int(ci.size), "rp": digest(rp, "rp"), "ci": digest(ci, "ci"),
         "w": digest(w, "w"), "color": digest(color, "color")}
    if agg is not None:
        d["agg"] = digest(agg, "agg")
        d["mate"] = digest(mate, "mate")
    return d


def main():
    cfg, prefix = int(sys.argv[1]), sys.argv[2]
    import graphgen as gg
    import oracle
    t0 = time.time()
    g = gg.config(cfg)
    G = oracle.Graph.from_csr(g.n, g.rp, g.ci, g.w)
    del g
    levels = oracle.build_hierarchy(G, oracle.Config())
    t1 = time.time()
    dig = []
    for ell, L in enumerate(levels):
        last = ell == len(levels) - 1
        dig.append(level_digests(L.g.rp, L.g.ci, L.g.w, L.color, None if last else L.q,
                                 None if last else L.mate))
    res = oracle.solve(G, oracle.Config(), levels=levels)
    t2 = time.time()
    np.save(prefix + ".vec.npy", res.vector)
    with open(prefix + ".json.tmp", "w") as f:
        json.dump({"config": cfg, "lambda2": res.lambda2, "residual_norm": res.residual_norm,
                   "num_levels": len(levels), "levels": dig,
                   "setup_s": t1 - t0, "solve_s": t2 - t1}, f)
    os.replace(prefix + ".json.tmp", prefix + ".json")


if __name__ == "__main__":
    main()
