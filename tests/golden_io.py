"""Load the committed golden fixtures (tests/golden/, made by make_golden.py from the reference)."""

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def arrays():
    return dict(np.load(os.path.join(GOLDEN, "golden_arrays.npz")))


@functools.lru_cache(maxsize=1)
def _json():
    with open(os.path.join(GOLDEN, "golden_digests.json")) as fh:
        return json.load(fh)


def digests():
    return _json()["digests"]


def meta():
    return _json()["meta"]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = a + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


SMALL = ("single_bottleneck", "shared_edge2", "shared_edge3", "chain", "diamond")
INCIDENCE = ("kept_rows", "demand", "com_path_ptr", "path_com", "hops", "pair_ptr", "pair_edge",
             "pair_path", "edge_path_count", "edge_pair_ptr", "edge_pairs")
STATE = ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg",
         "slack_demand", "slack_capacity")


def flat_inputs(prefix):
    A = arrays()
    return {k: A[f"{prefix}/in/{k}"] for k in
            ("capacity", "demand0", "com_path_ptr0", "path_edge_ptr0", "path_edges0")}


def kernel_seed(tag):
    if tag.startswith("small/"):
        return 100 + len(tag.split("/", 1)[1])
    return 5


@functools.lru_cache(maxsize=1)
def dao():
    """Drift-carry vectors (tests/golden/make_golden_dao.py): {tag: {case: arrays}}."""
    z = dict(np.load(os.path.join(GOLDEN, "golden_dao.npz")))
    out = {}
    for k, v in z.items():
        _, rest = k.split("/", 1)
        tag, case, field = rest.rsplit("/", 2)
        out.setdefault(tag, {}).setdefault(case, {})[field] = v
    return out
