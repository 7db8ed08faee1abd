"""Multi-GPU plumbing of the EE decode step: model replicas over request shards.

SURVEY §8(e): requests are independent (each owns its KV slots), so N GPUs run
N replicas over disjoint request shards with no data-path collective.  The one
exchange is at a profiling boundary: the Performance History Table counters
(exit-layer histogram ``ExitHistogram`` pht.hpp:15-38, breach count, token
count, sum of -logprob — ``record_token`` pht.hpp:92-102) are summed across
replicas, after which every rank computes the same greedy depth
(``choose_depth`` pht.hpp:119-126) and scheduler decision (pure functions of
the merged table, policy.hpp:243, :341).

The reduction is NCCL inside libeeb (``eeb_profile_allreduce``) on the GPU
box; any ``allreduce(int64 array, float) -> (array, float)`` callable can be
passed instead (the CPU tests use torch.distributed over gloo).
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Sequence

import numpy as np


def shard(request_ids: Sequence[int], world: int, rank: int) -> list[int]:
    """Round-robin request sharding by request id (generator substreams are per
    request, generator.hpp:319-323, so a shard is reproducible on its own)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return [r for r in request_ids if r % world == rank]


@dataclasses.dataclass
class ProfileCounters:
    """One model's profiler counters over a profiling window."""

    exit_layers: tuple
    hist: np.ndarray = None          # int64 [n_exits], ExitHistogram::counts by head
    n_breached: int = 0
    tokens: int = 0
    sum_neg_logprob: float = 0.0     # PhtEntry::sum_neg_logprob (pht.hpp:47-68)

    def __post_init__(self):
        if self.hist is None:
            self.hist = np.zeros(len(self.exit_layers), np.int64)

    def add_step(self, step: dict) -> None:
        """Accumulate one decode step's device outputs (hist, n_breached, sum_logprob)."""
        self.hist += np.asarray(step["hist"], np.int64)
        self.n_breached += int(np.asarray(step["n_breached"]).reshape(-1)[0])
        self.tokens += int(np.asarray(step["hist"]).sum())
        self.sum_neg_logprob -= float(np.asarray(step["sum_logprob"]).reshape(-1)[0])

    def pack(self) -> tuple[np.ndarray, float]:
        return np.concatenate([self.hist, [self.n_breached, self.tokens]]).astype(np.int64), self.sum_neg_logprob

    def unpack(self, counters: np.ndarray, s: float) -> None:
        n = len(self.exit_layers)
        self.hist = np.asarray(counters[:n], np.int64).copy()
        self.n_breached, self.tokens = int(counters[n]), int(counters[n + 1])
        self.sum_neg_logprob = float(s)

    def allreduce(self, fn: Callable[[np.ndarray, float], tuple[np.ndarray, float]]) -> "ProfileCounters":
        c, s = self.pack()
        self.unpack(*fn(c, s))
        return self

    def perplexity(self) -> float:
        """PhtEntry::perplexity (pht.hpp:64-67)."""
        if self.tokens == 0:
            raise ZeroDivisionError("no tokens recorded")
        return float(np.exp(self.sum_neg_logprob / self.tokens))

    def choose_depth(self, num_layers: int, coverage_target: float) -> int:
        return choose_depth(self.exit_layers, self.hist, num_layers, coverage_target)


def choose_depth(exit_layers: Sequence[int], counts: Sequence[int], num_layers: int, coverage_target: float) -> int:
    """Shallowest exit whose cumulative fraction reaches the target, else the
    final layer (pht.hpp:119-126); DomainError cases raise ValueError."""
    if not 0.0 < coverage_target <= 1.0:
        raise ValueError("coverage_target must be in (0, 1]")
    total = int(np.sum(counts))
    if total == 0:
        raise ValueError("choose_depth on an empty histogram")
    cum = 0
    for layer, c in zip(exit_layers, counts):
        cum += int(c)
        if cum / total >= coverage_target:
            return int(layer)
    return int(num_layers)


def torch_allreduce(group=None):
    """``allreduce`` over a torch.distributed process group (gloo or nccl)."""
    import torch
    import torch.distributed as dist

    def fn(counters: np.ndarray, s: float):
        t = torch.from_numpy(np.asarray(counters, np.int64).copy())
        f = torch.tensor([s], dtype=torch.float64)
        dist.all_reduce(t, group=group)
        dist.all_reduce(f, group=group)
        return t.numpy(), float(f.item())

    return fn


def eeb_allreduce(ctx):
    """``allreduce`` through libeeb's NCCL communicator (eeb_profile_allreduce)."""
    return lambda counters, s: ctx.profile_allreduce(np.asarray(counters, np.int64), s)
