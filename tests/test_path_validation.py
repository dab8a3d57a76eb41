"""build_instance's path validation (model.py:183-203 _check_path) on the host:
the native OpenMP check (pf_validate_paths) decides, the vectorised code names
the first bad path with the reference's message (tests/test_model.py style).
No GPU needed: validation runs before any device work."""

import pytest

import paper_2605_01748_b200 as pf
from paper_2605_01748_b200.model import _validate_paths
from paper_2605_01748_b200.topology import CommodityTable, PathSet


def _topo():
    # A -> B -> C -> D, plus C -> A (edge 3) and B -> A (edge 4)
    return pf.build_topology([("A", "B", 10, 1), ("B", "C", 10, 1), ("C", "D", 10, 1), ("C", "A", 10, 1),
                              ("B", "A", 10, 1)])


def _check(coms, paths):
    topo = _topo()
    table = CommodityTable.from_commodities(topo, [pf.Commodity(s, d, dem) for s, d, dem in coms])
    _validate_paths(topo, table, PathSet.from_lists(paths).to_flat())


def test_valid_paths_pass():
    _check([("A", "D", 5.0), ("B", "C", 1.0)], [[(0, 1, 2)], [(1,)]])


@pytest.mark.parametrize("paths, msg", [
    ([[()]], "empty path"),
    ([[(0, 9)]], "edge id 9 out of range"),
    ([[(1, 2)]], "does not start at 'A'"),
    ([[(0, 1)]], "does not end at 'D'"),
    ([[(0, 2)]], "edges 0 and 2 are not adjacent"),
    ([[(0, 1, 3, 0, 1, 2)]], "repeated node, path not simple"),
])
def test_first_bad_path_message(paths, msg):
    with pytest.raises(pf.InputError, match=msg):
        _check([("A", "D", 5.0)], paths)


def test_first_bad_path_in_commodity_major_order():
    # commodity 0's second path is bad, commodity 1's first path too: commodity 0 is named
    with pytest.raises(pf.InputError, match=r"commodity A→D, path 1: edges 0 and 2 are not adjacent"):
        _check([("A", "D", 5.0), ("B", "A", 1.0)], [[(0, 1, 2), (0, 2)], [(1, 2)]])
