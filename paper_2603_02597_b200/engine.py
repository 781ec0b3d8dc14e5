"""Engine configuration and work counters.

`BlockConfig` and `PassCounters` keep the reference's fields and validation
(/root/reference/pkg/src/lanebpe/engines.py:40-65 and :77-97).  On the device
`lane_count` has no effect (the reference documents it as scheduling-only);
`max_seq_len` / `chunk_budget` keep their meaning as the chunking semantics of
the batch path.  PassCounters.passes is the number of merges, i.e. input bytes
minus output ids, the identity the reference's acceptance gate checks
(test_acceptance.py:363-376).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class BlockConfig:
    lane_count: int = 256
    max_seq_len: int = 8192
    chunk_budget: int | None = None

    def __post_init__(self):
        if self.chunk_budget is None:
            object.__setattr__(self, "chunk_budget", self.max_seq_len)
        if self.lane_count < 1:
            raise ValueError(f"lane_count must be >= 1, got {self.lane_count}")
        if self.max_seq_len < 2:
            raise ValueError(f"max_seq_len must be >= 2, got {self.max_seq_len}")
        if not 2 <= self.chunk_budget <= self.max_seq_len:
            raise ValueError(
                f"chunk_budget must be in [2, max_seq_len={self.max_seq_len}], got {self.chunk_budget}")


@dataclass
class PassCounters:
    passes: int = 0
    lookups: int = 0
    compaction_moves: int = 0
    buffer_allocations: int = 0

    def merge_from(self, other: "PassCounters") -> None:
        self.passes += other.passes
        self.lookups += other.lookups
        self.compaction_moves += other.compaction_moves
        self.buffer_allocations += other.buffer_allocations
