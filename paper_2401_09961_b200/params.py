"""Parameter, trace and result types of the unwrap API.

Same names, fields, defaults and validation as the reference
(objective.py:30-41, irls.py:43-129) so a caller can switch packages.  These
are host-side records; no arithmetic on the data path lives here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class ModelParams:
    """objective.py:30-41 — quadratic-penalty strength tau, smoothing floor delta."""

    tau: float = 1e-2
    delta: float = 1e-6

    def __post_init__(self):
        if not (self.tau > 0 and math.isfinite(self.tau)):
            raise ValueError(f"tau must be positive and finite, got {self.tau}")
        if not (self.delta > 0 and math.isfinite(self.delta)):
            raise ValueError(f"delta must be positive and finite, got {self.delta}")


@dataclass(frozen=True)
class IrlsParams:
    """irls.py:43-64 — outer-loop and CG-budget controls."""

    max_iter_cg_start: int = 5
    rel_improvement_tol: float = 1e-3
    cg_growth_factor: float = 1.7
    max_outer_iters: int = 100
    max_cg_iters_cap: int = 10_000
    cg_rel_tol: float = 1e-10

    def __post_init__(self):
        checks = (
            (self.max_iter_cg_start < 1, "max_iter_cg_start must be >= 1"),
            (self.rel_improvement_tol <= 0, "rel_improvement_tol must be positive"),
            (self.cg_growth_factor <= 1, "cg_growth_factor must exceed 1"),
            (self.max_outer_iters < 1, "max_outer_iters must be >= 1"),
            (self.max_cg_iters_cap < self.max_iter_cg_start, "max_cg_iters_cap must be >= max_iter_cg_start"),
            (self.cg_rel_tol < 0, "cg_rel_tol must be >= 0"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)


@dataclass(frozen=True)
class IterationRecord:
    """irls.py:67-75 — one outer iteration of the trace."""

    k: int
    m_cg: int
    delta_rel: float | None
    h_delta: float
    cg_iters: int
    sufficient_decrease: bool
    fallback_used: bool


@dataclass
class IrlsTrace:
    """irls.py:78-92."""

    records: list = field(default_factory=list)

    def append(self, record):
        self.records.append(record)

    def h_values(self):
        return [r.h_delta for r in self.records]

    def fallback_count(self):
        return sum(1 for r in self.records if r.fallback_used)

    def __len__(self):
        return len(self.records)


@dataclass(frozen=True)
class BudgetDecision:
    """irls.py:95-100 — "keep", "stop" or "grow" with the budget going forward."""

    action: str
    m_cg: int


@dataclass(frozen=True)
class UnwrapResult:
    """irls.py:103-108 — mean-zero u and the slack fields, plus the trace."""

    u: np.ndarray
    vv: np.ndarray
    vh: np.ndarray
    trace: IrlsTrace


def relative_improvement(h_old_w, h_new_w):
    """irls.py:111-115."""
    if h_old_w <= 0:
        raise ValueError(f"reference objective value must be positive, got {h_old_w}")
    return (h_old_w - h_new_w) / h_old_w


def cg_budget_update(delta_rel, m_prev, m_prev2, params: IrlsParams):
    """irls.py:118-129 — keep while improving, stop after a fruitless grow, else grow."""
    if m_prev < 1:
        raise ValueError("m_prev must be >= 1")
    if delta_rel > params.rel_improvement_tol:
        return BudgetDecision("keep", m_prev)
    if m_prev != m_prev2 or m_prev >= params.max_cg_iters_cap:
        return BudgetDecision("stop", m_prev)
    return BudgetDecision("grow", min(math.ceil(params.cg_growth_factor * m_prev), params.max_cg_iters_cap))


def lipschitz_constant(c, p: ModelParams):
    """objective.py:103-105 — 12/tau + c_max^2/delta."""
    return 12.0 / p.tau + c.max_weight ** 2 / p.delta
