"""Wire formats for plans and gathered chains.

* Plans: ``plan_to_dict`` / ``plan_from_dict`` / ``save_plan`` / ``load_plan``
  follow ``pkg/src/swarmsched/plan.py:132-202`` (JSON, ``indent=2``,
  ``sort_keys=True``, trailing newline; ``ValueError`` naming the file for a
  malformed plan).
* Chains: ``chain_to_dict`` follows ``cli.py:106-117`` (``_chain_to_dict``) and
  ``chains_to_json`` the ``route --json`` payload ``{"chains": [...]}`` printed
  by ``_print_json`` (``cli.py:61-62``).
* ``chains_from_replay`` turns the device replay's per-layer GPU indices
  (``ss_replay*`` ``gpus`` output) into the reference's
  ``PipelineChain`` values: consecutive layers on one GPU merge into one
  ``LayerSlice`` hop exactly as ``router.py:188-194`` does, so a gathered
  device replay can be diffed line for line against ``swarmsched route --json``.
"""

from __future__ import annotations

import json
from typing import Iterable, List, Mapping, Sequence

import numpy as np

from .plan import AllocationPlan, PerKEntry, Pipeline, plan_to_dict
from .router import PipelineChain
from .topology import LayerSlice

__all__ = ["plan_to_dict", "plan_from_dict", "save_plan", "load_plan", "chain_to_dict", "chains_to_json",
           "chains_from_replay"]


def plan_from_dict(raw: Mapping) -> AllocationPlan:
    """Inverse of :func:`plan_to_dict` (plan.py:157-187)."""
    pipelines = tuple(
        Pipeline(stages=tuple(LayerSlice(gpu_id=str(s["gpu_id"]), start_layer=int(s["start_layer"]),
                                         end_layer=int(s["end_layer"])) for s in entry["stages"]),
                 region=entry.get("region"))
        for entry in raw["pipelines"])
    per_k = tuple(PerKEntry(region=str(e.get("region", "")), k=int(e["k"]), s_star=int(e["s_star"]),
                            z=float(e["z"])) for e in raw.get("per_k", []))
    return AllocationPlan(replication_count=int(raw["k"]), pipelines=pipelines,
                          stage_total=sum(p.stage_count for p in pipelines),
                          objective_score=float(raw["objective"]), per_k_table=per_k)


def save_plan(plan: AllocationPlan, path: str) -> None:
    """plan.py:190-193."""
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(plan_to_dict(plan), fh, indent=2, sort_keys=True)
        fh.write("\n")


def load_plan(path: str) -> AllocationPlan:
    """plan.py:196-202."""
    with open(path, "r", encoding="utf-8") as fh:
        raw = json.load(fh)
    try:
        return plan_from_dict(raw)
    except (TypeError, KeyError, AttributeError) as exc:
        raise ValueError(f"{path}: not a valid plan file ({exc})") from exc


def chain_to_dict(chain: PipelineChain) -> dict:
    """cli.py:106-117."""
    return {"hops": [{"gpu_id": h.gpu_id, "start_layer": h.start_layer, "end_layer": h.end_layer}
                     for h in chain.hops],
            "cost_s": chain.cost_s}


def chains_to_json(chains: Iterable[PipelineChain]) -> str:
    """The ``route --json`` payload (cli.py:159-161 with _print_json, 61-62)."""
    return json.dumps({"chains": [chain_to_dict(c) for c in chains]}, indent=2, sort_keys=True)


def chains_from_replay(ids: Sequence[str], gpus, costs) -> List[PipelineChain]:
    """PipelineChains of one scenario's replay.

    ``ids`` are the pool GPU ids in sorted order (the device GPU index space),
    ``gpus`` is ``[n_req, L]`` (the replay's ``gpus`` output row of one
    scenario), ``costs`` is ``[n_req]`` float64.  Hops merge consecutive layers
    served by one GPU (router.py:188-194); a GPU revisited later (A -> B -> A)
    starts a new hop, as in the reference.
    """
    g = np.asarray(gpus)
    c = np.asarray(costs, dtype=np.float64)
    if g.ndim != 2 or c.shape != (g.shape[0],):
        raise ValueError("gpus must be [n_req, L] and costs [n_req]")
    out = []
    for row, cost in zip(g.tolist(), c.tolist()):
        hops = []
        start = 1
        for layer in range(2, len(row) + 1):
            if row[layer - 1] != row[layer - 2]:
                hops.append(LayerSlice(ids[row[layer - 2]], start, layer - 1))
                start = layer
        hops.append(LayerSlice(ids[row[-1]], start, len(row)))
        out.append(PipelineChain(hops=tuple(hops), cost_s=float(cost)))
    return out
