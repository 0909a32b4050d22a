"""Multi-round FL driver around the C-ABI.

Argument marshalling and bookkeeping only: every round runs through ``fl_round``
(placement, packing, local SGD, FedAvg, NCCL reduce all inside libfl_b200.so), and
the Eq. 3 fit is the library's ``fl_lb_fit``.

* LB loop (§5): "The first FL round will use the naive
  round-robin strategy to collect data about client training time from all
  available workers" (L375); afterwards each GPU's records — (m, completion time)
  of every client it trained, collected with ``fl_set_timing_records`` — are fitted
  to Eq. 3 (L378-382) and the next round places clients with one fit per GPU
  (``FL_PLACE_LB_GPU``: workers fastest-first by the predicted time of the cohort's
  largest client, L385-386).  All records are kept (L434); ``window`` keeps only the
  last W rounds ("a time window for deleting older data", L437).
* Cohort sampling (reading A19): uniform without replacement from a seeded PCG64,
  one cohort per round, an input to ``fl_round`` (selection is separate from the
  round).
"""
from __future__ import annotations

from collections import deque

import numpy as np

from . import fl_lb_fit

_FIT_MIN_RECORDS = 4  # Eq. 3 has 4 parameters; fewer -> keep the bootstrap policy


def sample_cohort(n_clients: int, k: int, seed: int, round_index: int) -> np.ndarray:
    """k distinct client ids drawn uniformly without replacement, keyed (seed, round)."""
    rng = np.random.Generator(np.random.PCG64([seed, 1, round_index]))
    return np.sort(rng.choice(n_clients, size=k, replace=False)).astype(np.int64)


class RoundDriver:
    """Runs rounds on one rank's ctx.  ``policy`` in {"bu", "rr", "srr", "lb"};
    "lb" is the paper's learning-based loop (RR bootstrap, then per-GPU Eq. 3 fits)."""

    def __init__(self, ctx, policy: str = "bu", window: int | None = None, allgather=None):
        self.ctx = ctx
        self.policy = policy
        self.world = ctx.cfg.world_size
        self.allgather = allgather  # callable(np.ndarray[4]) -> np.ndarray[world, 4]; None = single rank
        self.records: deque = deque(maxlen=window)  # one (m[], t_ms[]) pair per round
        self.coef = None   # [world][4] fits used for the last LB placement
        self.kinds = None
        self.history = []  # per round: (policy used, stats)
        if policy == "lb":
            ctx.fl_set_timing_records(True)

    def _fit_all(self):
        m = np.concatenate([r[0] for r in self.records]) if self.records else np.zeros(0)
        t = np.concatenate([r[1] for r in self.records]) if self.records else np.zeros(0)
        if len(m) >= _FIT_MIN_RECORDS:
            coef, kind, _ = fl_lb_fit(m.astype(np.float64), t)
        else:  # a rank with too few records (e.g. no clients yet): a neutral unit-slope line
            coef, kind = np.array([1.0, 0.0, 1.0, 0.0]), -1
        if self.world > 1:
            if self.allgather is None:
                raise RuntimeError("RoundDriver: world_size > 1 needs an allgather for the per-GPU fits")
            allc = np.asarray(self.allgather(np.asarray(coef, np.float64)), np.float64).reshape(self.world, 4)
        else:
            allc = np.asarray(coef, np.float64).reshape(1, 4)
        return allc, kind

    def run(self, cohort, round_index: int):
        pol, coef = self.policy, None
        if self.policy == "lb":
            if round_index == 0 or not self.records:
                pol = "rr"  # L375: the first round is round-robin, to collect timing data
            else:
                self.coef, self.kinds = self._fit_all()
                pol, coef = "lb_gpu", self.coef
        stats = self.ctx.fl_round(cohort, policy=pol, lb_coef=coef, round_index=round_index)
        if self.world > 1 and self.allgather is not None:
            # "timedelta workers": slowest minus fastest rank's training time this round
            tr = np.asarray(self.allgather(np.array([stats["train_ms"], 0.0, 0.0, 0.0])), np.float64).reshape(-1, 4)
            stats["timedelta_ms"] = float(tr[:, 0].max() - tr[:, 0].min())
        else:
            stats["timedelta_ms"] = 0.0
        if self.policy == "lb":
            _, m, t = self.ctx.fl_get_client_times()
            self.records.append((m.astype(np.float64), t))
        self.history.append((pol, stats))
        return stats
