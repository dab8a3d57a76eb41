"""KSP gate at scale: digests of the reference's own
``harness.k_shortest_paths`` (networkx Yen, harness.py:138-176) over

* ALL 249,500 commodities of config 2 (random_topology(500, seed=500), k=8),
  in chunks of 2,500 commodities (one digest per chunk, so a mismatch names
  its chunk), and
* a 10,000-commodity sample of config 3 (random_topology(2000, seed=2000),
  k=8; commodity indices drawn with default_rng(11) from the 3,998,000
  ordered pairs in the reference's gravity order).

Run HERE (the build container) where the reference can be imported; about
15 minutes on 8 processes:

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_ksp.py

Output: tests/golden/golden_ksp.json.  Nothing here is read by the product;
tests/test_generators.py compares the native generator (csrc/ksp.cpp) against it.
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
OUT = os.path.dirname(os.path.abspath(__file__))
CHUNK = 2500


def _flat(path_set):
    cpp = [0]
    pep = [0]
    pe = []
    for paths in path_set.paths:
        cpp.append(cpp[-1] + len(paths))
        for p in paths:
            pe.extend(p)
            pep.append(len(pe))
    return (np.array(cpp, np.int64), np.array(pep, np.int64), np.array(pe, np.int64))


def digest_flat(cpp, pep, pe) -> str:
    """sha256 over the three CSR arrays as int64 (chunk-local offsets)."""
    h = hashlib.sha256()
    for a in (cpp, pep, pe):
        h.update(np.ascontiguousarray(a, np.int64).tobytes())
    return h.hexdigest()[:32]


_G = {}


def _init(n):
    from pathfair import harness
    topo = harness.random_topology(n, seed=n)
    _G["topo"] = topo
    _G["coms"] = harness.gravity_demands(topo, 1.0)


def _work(args):
    from pathfair import harness
    idx, k = args
    sub = [_G["coms"][i] for i in idx]
    ps = harness.k_shortest_paths(_G["topo"], sub, k)
    cpp, pep, pe = _flat(ps)
    return digest_flat(cpp, pep, pe), int(cpp[-1]), int(pe.size)


def run(n, k, chunks, procs):
    with mp.get_context("fork").Pool(procs, initializer=_init, initargs=(n,)) as pool:
        return pool.map(_work, [(c, k) for c in chunks], chunksize=1)


def main():
    procs = int(os.environ.get("PROCS", os.cpu_count() or 8))
    out = {"chunk": CHUNK, "k": 8}
    t = time.perf_counter()
    C2 = 500 * 499
    chunks = [np.arange(s, min(C2, s + CHUNK)) for s in range(0, C2, CHUNK)]
    res = run(500, 8, chunks, procs)
    out["cfg2"] = {"commodities": C2, "digests": [r[0] for r in res], "paths": sum(r[1] for r in res),
                   "pairs": sum(r[2] for r in res), "seconds": time.perf_counter() - t}
    print(f"cfg2 done in {time.perf_counter() - t:.0f}s", flush=True)
    t = time.perf_counter()
    C3 = 2000 * 1999
    pick = np.sort(np.random.default_rng(11).choice(C3, 10000, replace=False))
    chunks3 = [pick[s:s + 500] for s in range(0, pick.size, 500)]
    res = run(2000, 8, chunks3, procs)
    out["cfg3_sample"] = {"commodities_total": C3, "seed": 11, "size": int(pick.size), "chunk": 500,
                          "digests": [r[0] for r in res], "paths": sum(r[1] for r in res),
                          "pairs": sum(r[2] for r in res), "seconds": time.perf_counter() - t}
    print(f"cfg3 sample done in {time.perf_counter() - t:.0f}s", flush=True)
    with open(os.path.join(OUT, "golden_ksp.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
