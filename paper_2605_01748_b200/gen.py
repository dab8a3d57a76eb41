"""Synthetic input generation as a separate step: topology,
gravity demands and k shortest paths, written to one .npz.

    python -m paper_2605_01748_b200.gen --nodes 500 --k 8 --volume 1.5 --out data/cfg2.npz

random_topology / gravity_table follow the reference's generators bitwise
(harness.py:179-239) and k_shortest_paths its path rule (harness.py:138-176,
native host code in libpf_gen.so).  This module loads only the host
generator library -- never the GPU solver -- so a program that just needs
inputs (bench.py's reference arm) can run it in a subprocess and read the file.

File keys: capacity [E], demand [C0], cpp [C0+1], pep [P0+1], pe [NP0] (the
flat path set), and nodes / k / volume for identification.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np


def generate(nodes: int, k: int, volume_fraction: float):
    from .harness import gravity_table, k_shortest_paths, random_topology
    topo = random_topology(nodes, seed=nodes)
    tab = gravity_table(topo, volume_fraction * float(topo.capacity.sum()))
    flat = k_shortest_paths(topo, tab, k)
    return topo, tab, flat


def write(path: str, nodes: int, k: int, volume_fraction: float, topo, tab, flat) -> None:
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    tmp = f"{path}.{os.getpid()}.tmp.npz"  # atomic: concurrent writers may race
    np.savez(tmp, capacity=np.asarray(topo.capacity, np.float64), demand=np.asarray(tab.demand, np.float64),
             cpp=flat.com_path_ptr, pep=flat.path_edge_ptr, pe=flat.path_edges,
             nodes=np.int64(nodes), k=np.int64(k), volume=np.float64(volume_fraction))
    os.replace(tmp, path)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, required=True)
    ap.add_argument("--k", type=int, required=True)
    ap.add_argument("--volume", type=float, required=True, help="total demand as a fraction of total capacity")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    t = time.perf_counter()
    topo, tab, flat = generate(a.nodes, a.k, a.volume)
    write(a.out, a.nodes, a.k, a.volume, topo, tab, flat)
    print(f"[gen] {a.out}: {len(tab)} commodities, {flat.path_edge_ptr.shape[0] - 1} paths, "
          f"{flat.path_edges.shape[0]} pairs in {time.perf_counter() - t:.1f}s", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
