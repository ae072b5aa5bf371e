"""Configuration selection by single-source shortest path (section 6.1).

The paper builds a directed graph from the operators' dataflow: "Beginning from the input
data and proceeding in a topological order, we add a node to the graph for each input and
output data layout of the operator.  An edge is added from the input to the output layout,
weighted with the minimum runtime of any configuration with that layout ... We then run a
single-source shortest-path (SSSP) algorithm from the input to the output in the graph; the
resulting path gives our final configuration ... The path is saved to a configuration
file".  Here the operators are the stages of the layer step, the configurations
are the library's per-stage alternatives (enc_set_option knobs) measured on the B200, and a
layout names what a stage leaves in HBM for its consumers (e.g. Q, K, V in place in the QKV
tensor vs permuted [3, B, H, J, P]; P plus 1-bit keep words vs P and A).  Difference from the
paper (R21): the forward and backward chains are joined (the backward consumes the
forward's saved layouts), which the paper omits -- so every path is realizable.

Host-side, offline; no CUDA.  The graph is a DAG ordered by stage index, so SSSP is one
topological sweep (linear time).  Ties: lexicographically smallest config-id sequence.
"""
from __future__ import annotations

import itertools
import json
from dataclasses import asdict, dataclass, field


@dataclass(frozen=True)
class OpConfig:
    """One costed configuration of one operator (stage): consumes `in_layout`, produces
    `out_layout`, takes `cost_us`; `knobs` are the library options it needs."""
    op: str
    config_id: str
    in_layout: str
    out_layout: str
    cost_us: float
    knobs: tuple = ()


@dataclass
class SelectionGraph:
    ops: list
    source: str
    sink: str | None
    # edges[i][(in, out)] = the cheapest OpConfig of op i with those layouts
    edges: list = field(default_factory=list)

    def nodes(self):
        out = set()
        for i, e in enumerate(self.edges):
            for (a, b) in e:
                out.add((i, a))
                out.add((i + 1, b))
        return out


class SelectionError(ValueError):
    pass


def cost_table(rows):
    """Keep the minimum cost per (op, config_id, in, out); reject non-positive costs."""
    best = {}
    for c in rows:
        if not (c.cost_us > 0):
            raise SelectionError(f"non-positive cost for {c.op}/{c.config_id}")
        k = (c.op, c.config_id, c.in_layout, c.out_layout)
        if k not in best or c.cost_us < best[k].cost_us:
            best[k] = c
    return list(best.values())


def _better(a, b):
    """a strictly preferable to b (cost, then lexicographic config ids)."""
    if b is None:
        return True
    if a[0] != b[0]:
        return a[0] < b[0]
    return a[1] < b[1]


def build_selection_graph(ops, configs, source, sink=None):
    """Edges per operator from the input to the output layout, weighted with the minimum
    cost of any configuration with those layouts; only configurations with at least
    one input and one output edge are kept: forward reachability from `source`,
    backward reachability to `sink` (any layout when sink is None)."""
    by_op = {o: [] for o in ops}
    for c in cost_table(configs):
        if c.op not in by_op:
            raise SelectionError(f"unknown operator {c.op}")
        by_op[c.op].append(c)
    for o in ops:
        if not by_op[o]:
            raise SelectionError(f"operator {o} has no costed configuration")
    edges = []
    for o in ops:
        e = {}
        for c in sorted(by_op[o], key=lambda c: (c.cost_us, c.config_id)):
            k = (c.in_layout, c.out_layout)
            if k not in e:
                e[k] = c
        edges.append(e)
    # prune: reachable from the source, and able to reach the sink
    reach = {source}
    for i, e in enumerate(edges):
        edges[i] = {k: c for k, c in e.items() if k[0] in reach}
        reach = {k[1] for k in edges[i]}
    alive = reach if sink is None else ({sink} & reach)
    for i in reversed(range(len(edges))):
        edges[i] = {k: c for k, c in edges[i].items() if k[1] in alive}
        alive = {k[0] for k in edges[i]}
    return SelectionGraph(list(ops), source, sink, edges)


def select_configuration(sg):
    """DAG SSSP in one topological sweep; returns (configs along the path, total cost)."""
    dist = {sg.source: (0.0, ())}
    back = [dict() for _ in sg.edges]
    for i, e in enumerate(sg.edges):
        nd = {}
        for (a, b), c in sorted(e.items()):
            if a not in dist:
                continue
            cand = (dist[a][0] + c.cost_us, dist[a][1] + (c.config_id,))
            if _better(cand, nd.get(b)):
                nd[b] = cand
                back[i][b] = (a, c)
        dist = nd
    if not dist or (sg.sink is not None and sg.sink not in dist):
        raise SelectionError("sink unreachable: no layout-compatible chain")
    end = sg.sink if sg.sink is not None else min(dist, key=lambda k: (dist[k][0], dist[k][1]))
    path, node = [], end
    for i in reversed(range(len(sg.edges))):
        a, c = back[i][node]
        path.append(c)
        node = a
    path.reverse()
    return path, dist[end][0]


def brute_force(ops, configs, source, sink=None):
    """Exhaustive minimum over all layout-consistent configuration tuples (test oracle)."""
    by_op = {o: [c for c in cost_table(configs) if c.op == o] for o in ops}
    best = None
    for tup in itertools.product(*[by_op[o] for o in ops]):
        if tup[0].in_layout != source:
            continue
        if any(tup[i].out_layout != tup[i + 1].in_layout for i in range(len(tup) - 1)):
            continue
        if sink is not None and tup[-1].out_layout != sink:
            continue
        cand = (sum(c.cost_us for c in tup), tuple(c.config_id for c in tup))
        if _better(cand, best):
            best = cand
            best_t = tup
    if best is None:
        raise SelectionError("no layout-compatible chain")
    return list(best_t), best[0]


def knobs_of(path):
    """Merged option settings of a path; raises if two configurations disagree."""
    out = {}
    for c in path:
        for k, v in c.knobs:
            if out.setdefault(k, v) != v:
                raise SelectionError(f"conflicting knob {k} along the path")
    return out


def emit_configuration(path, total, fname, extra=None):
    """The configuration file: the chosen configuration per operator + knobs."""
    doc = {"total_us": total, "knobs": knobs_of(path),
           "path": [dict(asdict(c), knobs=list(map(list, c.knobs))) for c in path]}
    if extra:
        doc.update(extra)
    with open(fname, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)


def load_configuration(fname):
    with open(fname) as f:
        doc = json.load(f)
    path = [OpConfig(p["op"], p["config_id"], p["in_layout"], p["out_layout"], p["cost_us"],
                     tuple(tuple(k) for k in p["knobs"])) for p in doc["path"]]
    return path, doc["total_us"], doc["knobs"]
