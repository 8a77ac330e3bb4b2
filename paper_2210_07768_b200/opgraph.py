"""Call-graph expansion and the layer schedule (host, once per run).

Same semantics as the reference ``pkg/src/featurebox/opgraph.py``:
``expand_call_graph`` (:114-200) turns every operator into one body node plus
one node per pre/post call; ``layer_schedule`` (:265-292) puts each node one
layer past its deepest predecessor, name-sorted within a layer.

On the B200 every node is placed on the device -- dictionary lookups included
(they are HBM hash tables) -- so ``place_operators`` keeps
the reference signature but never creates host nodes or H2D transfer nodes.
The layers become the evaluation order inside one fused kernel per driver
chunk: all operators are row-local, so a layer barrier of the reference
(device.py:405-409) is the program order of a row's thread.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

from .featureops import FeatureConfigError, FunctionRef, OperatorSpec

DEVICE = "device"
HOST = "host"
BODY, PRE, POST = "body", "pre", "post"


class CycleError(ValueError):
    """The operator dependency graph contains a cycle (opgraph.py:27)."""


class InvalidPlanError(ValueError):
    pass


@dataclass(frozen=True)
class Node:
    name: str
    role: str
    op: str
    func: FunctionRef
    footprint_bytes: int
    kind: str
    reads: tuple[str, ...] = ()
    writes: tuple[str, ...] = ()
    slot: int | None = None
    out_index: int | None = None


@dataclass
class OperatorDag:
    nodes: dict[str, Node]
    edges: tuple[tuple[str, str], ...]
    col_producer: dict[str, str]

    def __post_init__(self):
        preds: dict[str, list[str]] = {n: [] for n in self.nodes}
        succs: dict[str, list[str]] = {n: [] for n in self.nodes}
        for u, v in self.edges:
            preds[v].append(u)
            succs[u].append(v)
        self.preds = {n: tuple(sorted(p)) for n, p in preds.items()}
        self.succs = {n: tuple(sorted(s)) for n, s in succs.items()}

    def external_inputs(self) -> tuple[str, ...]:
        read = {c for node in self.nodes.values() for c in node.reads}
        return tuple(sorted(read - set(self.col_producer)))


def _cycle(dag_nodes, succs) -> list[str]:
    state: dict[str, int] = {}
    path: list[str] = []

    def visit(u):
        state[u] = 1
        path.append(u)
        for v in succs.get(u, ()):
            if state.get(v) == 1:
                return path[path.index(v):] + [v]
            if not state.get(v):
                found = visit(v)
                if found:
                    return found
        path.pop()
        state[u] = 2
        return None

    for n in sorted(dag_nodes):
        if not state.get(n):
            found = visit(n)
            if found:
                return found
    return []


def expand_call_graph(specs: Sequence[OperatorSpec]) -> OperatorDag:
    names = [s.name for s in specs]
    if len(set(names)) != len(names):
        dup = sorted({n for n in names if names.count(n) > 1})
        raise FeatureConfigError(f"duplicate operator names: {dup}")
    nodes: dict[str, Node] = {}
    edges: set[tuple[str, str]] = set()
    producer: dict[str, str] = {}

    def add(node: Node):
        nodes[node.name] = node
        for c in node.writes:
            if c in producer:
                raise FeatureConfigError(
                    f"output column {c!r} produced by both {producer[c]!r} and {node.name!r}")
            producer[c] = node.name

    for spec in specs:
        pre_slots = {spec.pre_slot(i) for i in range(len(spec.pre_calls))}
        add(Node(spec.name, BODY, spec.name, spec.body, spec.footprint_bytes, spec.kind,
                 tuple(c for i, c in enumerate(spec.inputs) if i not in pre_slots),
                 () if spec.post_calls else spec.outputs))
        for i, ref in enumerate(spec.pre_calls):
            slot = spec.pre_slot(i)
            nm = f"{spec.name}.pre{i + 1}"
            add(Node(nm, PRE, spec.name, ref, ref.footprint_bytes, ref.kind,
                     (spec.inputs[slot],), (), slot=slot))
            edges.add((nm, spec.name))
        for j, ref in enumerate(spec.post_calls):
            nm = f"{spec.name}.post{j + 1}"
            add(Node(nm, POST, spec.name, ref, ref.footprint_bytes, ref.kind,
                     (), (spec.outputs[j],), out_index=j))
            edges.add((spec.name, nm))
    for node in nodes.values():
        for c in node.reads:
            if c in producer:
                edges.add((producer[c], node.name))
    dag = OperatorDag(nodes, tuple(sorted(edges)), producer)
    cyc = _cycle(dag.nodes, dag.succs)
    if cyc:
        raise CycleError("dependency cycle: " + " -> ".join(cyc))
    return dag


@dataclass(frozen=True)
class LayerPlan:
    layers: tuple[tuple[str, ...], ...]
    placement: Mapping[str, str] = field(default_factory=dict)
    transfers: tuple = ()

    @property
    def layer_of(self) -> dict[str, int]:
        return {n: i + 1 for i, layer in enumerate(self.layers) for n in layer}

    def device_nodes(self, layer_index: int) -> tuple[str, ...]:
        return tuple(n for n in self.layers[layer_index - 1]
                     if self.placement.get(n, DEVICE) == DEVICE)

    def node_order(self) -> list[tuple[int, str]]:
        """(layer, name) in evaluation order: the fused kernel's program order."""
        return [(i + 1, n) for i, layer in enumerate(self.layers) for n in layer]


def layer_schedule(dag: OperatorDag) -> LayerPlan:
    """Longest-path depth from the sources (opgraph.py:265-292)."""
    indeg = {n: len(dag.preds[n]) for n in dag.nodes}
    ready = sorted(n for n, d in indeg.items() if d == 0)
    depth = {n: 1 for n in ready}
    seen = 0
    while ready:
        u = ready.pop()
        seen += 1
        for v in dag.succs[u]:
            depth[v] = max(depth.get(v, 1), depth[u] + 1)
            indeg[v] -= 1
            if indeg[v] == 0:
                ready.append(v)
                ready.sort()
    if seen != len(dag.nodes):
        raise CycleError("dependency cycle: " + " -> ".join(_cycle(dag.nodes, dag.succs)))
    n_layers = max(depth.values(), default=0)
    buckets: list[list[str]] = [[] for _ in range(n_layers)]
    for n, d in depth.items():
        buckets[d - 1].append(n)
    return LayerPlan(tuple(tuple(sorted(b)) for b in buckets))


@dataclass(frozen=True)
class PlacementBudget:
    device_memory_bytes: int | float

    def __post_init__(self):
        if not self.device_memory_bytes > 0:
            raise ValueError("device_memory_bytes must be positive")


def place_operators(plan: LayerPlan, budget: PlacementBudget | None,
                    dag: OperatorDag) -> LayerPlan:
    """Every node on the device; no host nodes, no H2D transfer nodes."""
    placed = LayerPlan(plan.layers, {n: DEVICE for n in dag.nodes}, ())
    validate_plan(placed, dag)
    return placed


def reference_placement(dag: OperatorDag, budget_bytes: int | float) -> dict[str, str]:
    """Where the REFERENCE would run each node: host iff its footprint exceeds the
    device budget (opgraph.py:295-324).  The B200 runs every node on the device,
    but two results depend on this: which token calls draw from the reference's
    arena pool (device.py:328-338) and which failure a layer reports first --
    its device nodes in name order, then its host nodes (device.py:362-406)."""
    return {n: HOST if nd.footprint_bytes > budget_bytes else DEVICE
            for n, nd in dag.nodes.items()}


def reference_node_order(plan: LayerPlan, placement: Mapping[str, str]) -> list[tuple[int, str]]:
    """(layer, name) in the reference's failure-precedence order: per layer the
    device nodes by name, then the host nodes by name."""
    return [(i + 1, n) for i, layer in enumerate(plan.layers)
            for n in sorted(layer, key=lambda m: (placement[m] != DEVICE, m))]


def validate_plan(plan: LayerPlan, dag: OperatorDag) -> None:
    layer_of = plan.layer_of
    if set(layer_of) != set(dag.nodes):
        raise InvalidPlanError("plan nodes differ from dag nodes")
    for u, v in dag.edges:
        if layer_of[u] >= layer_of[v]:
            raise InvalidPlanError(f"edge {u}->{v} not strictly layered")
    for n in dag.nodes:
        want = 1 + max((layer_of[p] for p in dag.preds[n]), default=0)
        if layer_of[n] != want:
            raise InvalidPlanError(f"{n}: layer {layer_of[n]}, longest-path depth {want}")


def fused_launch_count(plan: LayerPlan) -> int:
    """Launches per driver chunk on the B200 engine: the whole plan is one."""
    return 1 if plan.layers else 0


def plan_report(plan: LayerPlan, dag: OperatorDag) -> str:
    lines = [f"plan: {len(dag.nodes)} operators, {len(plan.layers)} layers, "
             f"1 fused kernel per chunk (all nodes on device)"]
    for i, layer in enumerate(plan.layers, 1):
        lines.append(f"layer {i}: " + ", ".join(
            f"{n} ({dag.nodes[n].func.spec}) [device]" for n in layer))
    return "\n".join(lines)
