"""Loader for tests/golden/reference_runs.{npz,json} (see make_golden.py)."""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class GoldenRun:
    graph: str
    n: int
    undirected: bool
    src: np.ndarray
    dst: np.ndarray
    app: str
    kwargs: dict
    values: np.ndarray
    superstep_count: int
    hit_superstep_cap: bool
    active_counts: list
    messages_sent: list

    @property
    def id(self) -> str:
        kw = ",".join(f"{k}={v}" for k, v in sorted(self.kwargs.items()))
        return f"{self.graph}:{self.app}({kw})"


def load_runs() -> list[GoldenRun]:
    with open(os.path.join(_DIR, "reference_runs.json")) as fh:
        manifest = json.load(fh)
    arrays = np.load(os.path.join(_DIR, "reference_runs.npz"))
    out = []
    for ci, case in enumerate(manifest["cases"]):
        src = arrays[f"c{ci}_src"].astype(np.int64)
        dst = arrays[f"c{ci}_dst"].astype(np.int64)
        for run in case["runs"]:
            out.append(GoldenRun(case["name"], case["n"], case["undirected"],
                                 src, dst, run["app"], run["kwargs"],
                                 arrays[run["key"] + "_values"],
                                 run["superstep_count"],
                                 run["hit_superstep_cap"],
                                 run["active_counts"], run["messages_sent"]))
    return out


#: tests/test_algorithms.py:27-28 of the reference (10 steps, d = 0.85)
PATH3_RANKS = [0.271832724656722, 0.456334550686556, 0.271832724656722]
DANGLING_RANKS = [0.197582820658829, 0.281552611664937, 0.520864567676234]
