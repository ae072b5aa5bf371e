"""Configuration selection by SSSP (paper_2007_00072_b200/config_select.py)
against exhaustive enumeration of all layout-consistent configuration tuples (the test
oracle SPEC.md:401 names), plus the construction rules (min-over-matching-configs edge
weights, pruning of configurations without an input and an output edge)."""
import random

import pytest

from paper_2007_00072_b200.config_select import (OpConfig, SelectionError, brute_force,
                                                 build_selection_graph, cost_table,
                                                 emit_configuration, knobs_of,
                                                 load_configuration, select_configuration)


def C(op, cid, a, b, cost, knobs=()):
    return OpConfig(op, cid, a, b, cost, knobs)


def test_single_op_takes_cheapest():
    cfgs = [C("o", "x", "in", "L0", 5.0), C("o", "y", "in", "L1", 3.0)]
    path, tot = select_configuration(build_selection_graph(["o"], cfgs, "in"))
    assert [c.config_id for c in path] == ["y"] and tot == 3.0


def test_incompatible_local_optima():
    # op a: cheapest output L0; op b: cheapest consumes L1 -> the chain must trade off
    cfgs = [C("a", "a0", "in", "L0", 1.0), C("a", "a1", "in", "L1", 4.0),
            C("b", "b0", "L0", "M", 10.0), C("b", "b1", "L1", "M", 2.0),
            C("c", "c0", "M", "out", 1.0)]
    sg = build_selection_graph(["a", "b", "c"], cfgs, "in", "out")
    path, tot = select_configuration(sg)
    assert [c.config_id for c in path] == ["a1", "b1", "c0"] and tot == 7.0
    assert brute_force(["a", "b", "c"], cfgs, "in", "out")[1] == tot


def test_edge_weight_is_min_over_matching_configs_and_duplicates():
    cfgs = [C("a", "v1", "in", "L", 9.0), C("a", "v2", "in", "L", 4.0), C("a", "v2", "in", "L", 6.0)]
    assert len(cost_table(cfgs)) == 2
    sg = build_selection_graph(["a"], cfgs, "in")
    assert sg.edges[0][("in", "L")].cost_us == 4.0
    with pytest.raises(SelectionError):
        cost_table([C("a", "z", "in", "L", 0.0)])


def test_pruning_dead_ends():
    cfgs = [C("a", "a0", "in", "L0", 1.0), C("a", "dead", "in", "Lx", 0.5),
            C("b", "b0", "L0", "out", 1.0)]
    sg = build_selection_graph(["a", "b"], cfgs, "in", "out")
    assert ("in", "Lx") not in sg.edges[0]
    assert len(sg.nodes()) == 3


def test_unreachable_sink_and_missing_op():
    cfgs = [C("a", "a0", "in", "L0", 1.0), C("b", "b0", "L1", "out", 1.0)]
    with pytest.raises(SelectionError):
        select_configuration(build_selection_graph(["a", "b"], cfgs, "in", "out"))
    with pytest.raises(SelectionError):
        build_selection_graph(["a", "b", "c"], cfgs, "in")


@pytest.mark.parametrize("seed", range(40))
def test_random_dags_match_brute_force(seed):
    rng = random.Random(seed)
    nops, nl = rng.randint(1, 6), rng.randint(1, 4)
    ops = [f"op{i}" for i in range(nops)]
    cfgs = []
    for i, o in enumerate(ops):
        ins = ["in"] if i == 0 else [f"L{i}_{k}" for k in range(nl)]
        outs = [f"L{i + 1}_{k}" for k in range(nl)] if i + 1 < nops else ["out"]
        for j in range(rng.randint(1, 8)):
            # integer costs make exact ties frequent: the tie-break must agree too
            cfgs.append(C(o, f"{o}c{j}", rng.choice(ins), rng.choice(outs), float(rng.randint(1, 9))))
    try:
        want, wtot = brute_force(ops, cfgs, "in", "out")
    except SelectionError:
        with pytest.raises(SelectionError):
            select_configuration(build_selection_graph(ops, cfgs, "in", "out"))
        return
    path, tot = select_configuration(build_selection_graph(ops, cfgs, "in", "out"))
    assert tot == wtot
    assert [c.config_id for c in path] == [c.config_id for c in want]
    for a, b in zip(path, path[1:]):
        assert a.out_layout == b.in_layout


def test_emit_roundtrip_and_knob_conflicts(tmp_path):
    cfgs = [C("a", "a0", "in", "L", 1.0, (("attn_tc", 1),)), C("b", "b0", "L", "out", 2.0,
                                                                (("attn_bh", 0),))]
    path, tot = select_configuration(build_selection_graph(["a", "b"], cfgs, "in", "out"))
    f = tmp_path / "cfg.json"
    emit_configuration(path, tot, f)
    p2, t2, knobs = load_configuration(f)
    assert p2 == path and t2 == tot and knobs == {"attn_tc": 1, "attn_bh": 0}
    with pytest.raises(SelectionError):
        knobs_of([C("a", "x", "i", "o", 1.0, (("k", 1),)), C("b", "y", "o", "p", 1.0, (("k", 0),))])
