"""Sharding-plan ingest: the reference planner's output, consumed unchanged.

Mirrors the plan types of neosim/planner.py:38-156 (``SchemeKind``,
``Scheme``, ``Shard``, ``TableAssignment``, ``ShardingPlan``,
``even_bounds``), its JSON document (planner.py:827-919 plan_to_json /
plan_from_json) and its invariants (planner.py:770-824 validate_plan).
Plans made by the reference's ``plan_4d`` / ``hierarchical_plan`` are
accepted directly (duck typing) or as their JSON.

``RankLayout`` turns a plan into what one GPU needs: its local shards in
plan order, their column offsets inside the pooled rows it produces, the
data-parallel tables it replicates, and the pooled-row column map.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

from .errors import InvalidScheme, InvalidValue, MalformedDocument, MissingKey


class SchemeKind(str, Enum):
    TABLE_WISE = "table_wise"
    ROW_WISE = "row_wise"
    COLUMN_WISE = "column_wise"
    DATA_PARALLEL = "data_parallel"


@dataclass(frozen=True)
class Scheme:
    kind: SchemeKind
    num_row_shards: int = 1
    col_splits: tuple = ()
    hierarchical: Optional[tuple] = None


@dataclass(frozen=True)
class Shard:
    worker: Optional[int]
    rows: Optional[tuple] = None
    cols: Optional[tuple] = None


@dataclass(frozen=True)
class TableAssignment:
    table_id: str
    scheme: Scheme
    shards: tuple


@dataclass(frozen=True)
class ShardingPlan:
    num_workers: int
    gpus_per_node: int
    assignments: tuple
    heuristic: str = "greedy"

    def assignment_for(self, table_id: str):
        for a in self.assignments:
            if a.table_id == table_id:
                return a
        raise KeyError(table_id)


def even_bounds(extent: int, parts: int) -> list:
    """[0, extent) in `parts` contiguous ranges; the first extent % parts
    ranges get one extra row (planner.py:148-156)."""
    q, r = divmod(extent, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + q + (i < r)
        out.append((lo, hi))
        lo = hi
    return out


def kind_of(assignment) -> str:
    k = assignment.scheme.kind
    return getattr(k, "value", k)


def plan_from_json(text: str) -> ShardingPlan:
    """Parse the reference's plan document (planner.py:827-919)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise MalformedDocument(f"not valid JSON: {exc}") from None
    if not isinstance(doc, dict):
        raise MalformedDocument("plan document must be an object")
    try:
        W = doc["num_workers"]
        out = []
        for td in doc["tables"]:
            sd = td["scheme"]
            scheme = Scheme(SchemeKind(sd["kind"]), num_row_shards=sd.get("num_row_shards", 1),
                            col_splits=tuple(tuple(p) for p in sd.get("col_splits", [])),
                            hierarchical=tuple(SchemeKind(v) for v in sd["hierarchical"])
                            if "hierarchical" in sd else None)
            shards = tuple(Shard(worker=s.get("worker"), rows=tuple(s["rows"]) if "rows" in s else None,
                                 cols=tuple(s["cols"]) if "cols" in s else None) for s in td["shards"])
            out.append(TableAssignment(td["table_id"], scheme, shards))
    except KeyError as exc:
        raise MissingKey(str(exc)) from None
    except (TypeError, ValueError) as exc:
        raise InvalidValue("plan", str(exc)) from None
    return ShardingPlan(W, doc.get("gpus_per_node", W), tuple(out), doc.get("heuristic", "greedy"))


def plan_to_json(plan) -> str:
    doc = {"spec_version": 1, "num_workers": plan.num_workers, "gpus_per_node": plan.gpus_per_node,
           "heuristic": getattr(plan, "heuristic", "greedy"), "tables": []}
    for a in plan.assignments:
        sd = {"kind": kind_of(a)}
        if sd["kind"] == "row_wise":
            sd["num_row_shards"] = a.scheme.num_row_shards
        if sd["kind"] == "column_wise":
            sd["col_splits"] = [list(p) for p in a.scheme.col_splits]
        if a.scheme.hierarchical:
            sd["hierarchical"] = [getattr(k, "value", k) for k in a.scheme.hierarchical]
        doc["tables"].append({"table_id": a.table_id, "scheme": sd, "shards": [
            {"worker": s.worker, **({"rows": list(s.rows)} if s.rows else {}),
             **({"cols": list(s.cols)} if s.cols else {})} for s in a.shards]})
    return json.dumps(doc, indent=2, sort_keys=True)


def validate_plan(plan, model) -> None:
    """Coverage and placement invariants (planner.py:770-824)."""
    by_id = {t.id: t for t in model.tables}
    seen = set()
    for a in plan.assignments:
        table = by_id.get(a.table_id)
        if table is None:
            raise InvalidScheme(f"plan names unknown table {a.table_id}")
        if a.table_id in seen:
            raise InvalidScheme(f"table {a.table_id} assigned twice")
        seen.add(a.table_id)
        kind = kind_of(a)
        for s in a.shards:
            if s.worker is not None and not 0 <= s.worker < plan.num_workers:
                raise InvalidScheme(f"{a.table_id}: worker {s.worker} out of range")
            if (s.worker is None) != (kind == "data_parallel"):
                raise InvalidScheme(f"{a.table_id}: replicated shard only valid for DP")
        if kind in ("row_wise", "column_wise"):
            attr, extent = ("rows", table.num_rows) if kind == "row_wise" else ("cols", table.dim)
            if any(getattr(s, attr) is None for s in a.shards):
                raise InvalidScheme(f"{a.table_id}: shard missing bounds")
            pos = 0
            for lo, hi in sorted(getattr(s, attr) for s in a.shards):
                if lo != pos or hi <= lo:
                    raise InvalidScheme(f"{a.table_id}: shards must tile [0, {extent})")
                pos = hi
            if pos != extent:
                raise InvalidScheme(f"{a.table_id}: shards must cover [0, {extent})")
        elif len(a.shards) != 1:
            raise InvalidScheme(f"{a.table_id}: expected a single shard")
    missing = set(by_id) - seen
    if missing:
        raise InvalidScheme(f"tables not assigned: {sorted(missing)}")


# ---------------------------------------------------------------------------
# per-rank layout


@dataclass
class LocalShard:
    """One non-DP shard placed on a rank."""

    table: int          # model table index
    table_id: str
    kind: str           # table_wise | row_wise | column_wise
    index: int          # shard index inside its assignment
    rows: tuple         # (r0, r1) of the full table
    cols: tuple         # (c0, c1)
    out_col: int = 0    # column offset in this rank's pooled rows

    @property
    def num_rows(self) -> int:
        return self.rows[1] - self.rows[0]

    @property
    def dim(self) -> int:
        return self.cols[1] - self.cols[0]


@dataclass
class RankLayout:
    """Everything rank-specific derived from (model, plan)."""

    world: int
    owned: list = field(default_factory=list)       # owned[v] = [LocalShard] on rank v, plan order
    dp_tables: list = field(default_factory=list)   # model indices of DP tables
    model_cols: list = field(default_factory=list)  # model column offset of each table
    total_dim: int = 0
    rw_bounds: dict = field(default_factory=dict)   # table -> sorted [(r0, r1)], shard index order
    rw_shard_of_bounds: dict = field(default_factory=dict)

    def width(self, v: int) -> int:
        return sum(s.dim for s in self.owned[v])

    @property
    def dp_dim(self) -> int:
        return sum(self.dims[t] for t in self.dp_tables)


def rank_layout(model, plan) -> RankLayout:
    validate_plan(plan, model)
    W = plan.num_workers
    lay = RankLayout(world=W, owned=[[] for _ in range(W)])
    lay.dims = [t.dim for t in model.tables]
    lay.rows = [t.num_rows for t in model.tables]
    lay.ids = [t.id for t in model.tables]
    col = 0
    for t in model.tables:
        lay.model_cols.append(col)
        col += t.dim
    lay.total_dim = col
    by_id = {a.table_id: a for a in plan.assignments}
    for ti, table in enumerate(model.tables):  # model order; shards in assignment order
        a = by_id[table.id]
        kind = kind_of(a)
        if kind == "data_parallel":
            lay.dp_tables.append(ti)
            continue
        if kind == "row_wise":
            lay.rw_bounds[ti] = sorted(tuple(s.rows) for s in a.shards)
        for i, s in enumerate(a.shards):
            rows = tuple(s.rows) if s.rows else (0, table.num_rows)
            cols = tuple(s.cols) if s.cols else (0, table.dim)
            lay.owned[s.worker].append(LocalShard(ti, table.id, kind, i, rows, cols))
    for v in range(W):
        c = 0
        for s in lay.owned[v]:
            s.out_col = c
            c += s.dim
    return lay
