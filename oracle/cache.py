"""Degree-ordered static device feature cache (oracle side).

Paper: transmission abstraction §3.2 P:260-273 ("the device cache is
initialized according to the available memory resource ... figures out which
part of the mini-batch has been cached ... the remaining part is filtered out
from the host"); PaGraph template = static cache with ratio r, update
disabled; cache volume r|V|; transfer
volume n_attr |V_i| (1-hit) (Eq.6).

Readings: Q7 capacity floor(r*|V|) in IEEE double, ties by lower id
(SPEC S:188); degree = stored CSR row length.  Q8 hit accounting per
unique input row of F_L.  Sharded placement over G GPUs:
owner = rank mod G, local slot = rank div G.
"""
from __future__ import annotations

import math

import numpy as np

POLICY_NONE = 0
POLICY_DEGREE = 1


def cache_capacity(ratio: float, n: int, policy: int = POLICY_DEGREE) -> int:
    """C = floor(ratio * |V|); policy NONE => 0."""
    if not (0.0 <= ratio <= 1.0) or math.isnan(ratio):
        raise ValueError("parameter error: ratio must be in [0,1]")
    if policy == POLICY_NONE:
        return 0
    return int(math.floor(float(ratio) * float(n)))


def degree_rank(indptr: np.ndarray) -> np.ndarray:
    """rank[v] = position of v in the order (degree desc, id asc)."""
    deg = np.diff(np.asarray(indptr, dtype=np.int64))
    n = deg.shape[0]
    ids = np.arange(n, dtype=np.int64)
    order = np.lexsort((ids, -deg))  # primary -deg, secondary id
    rank = np.empty(n, dtype=np.int64)
    rank[order] = ids
    return rank


def cache_slots(indptr: np.ndarray, ratio: float, policy: int = POLICY_DEGREE,
                world: int = 1):
    """Per vertex: (slot, owner, local_slot).  slot = rank if rank < C else -1.

    For G = world shards: owner = rank mod G, local_slot = rank div G
    (both -1 for uncached vertices)."""
    n = len(indptr) - 1
    C = cache_capacity(ratio, n, policy)
    rank = degree_rank(indptr)
    cached = rank < C
    slot = np.where(cached, rank, -1)
    owner = np.where(cached, rank % world, -1)
    local = np.where(cached, rank // world, -1)
    return slot, owner, local


def access_counts(slot: np.ndarray, owner: np.ndarray, rows: np.ndarray, me: int = 0):
    """Counters over the unique rows F_L (Q8):
    hits = #{slot >= 0}; peer = #{hit and owner != me}; host misses = rows - hits."""
    rows = np.asarray(rows, dtype=np.int64)
    s = slot[rows]
    hit = s >= 0
    hits = int(hit.sum())
    peer = int((hit & (owner[rows] != me)).sum())
    return dict(rows=int(rows.size), hits=hits, hits_local=hits - peer, hits_peer=peer,
                misses_host=int(rows.size) - hits)


POLICY_FIFO = 2
POLICY_LRU = 3


class DynamicCache:
    """Dynamic cache with all-miss admission (SPEC
    S:181-219 access_batch; the paper's cache "updating" and the replaced
    volume of Eq.5).  Written as the plain sequential
    simulation of SPEC's access_batch:

      * the batch's rows are accessed; hits = rows resident, misses = rest;
      * LRU: every hit is stamped with the batch index t (FIFO: no change);
      * the misses are admitted one at a time in ascending F_L order (the
        order they appear in the batch), each stamped t and given the next
        admission sequence number; a free slot (lowest index first) is taken
        if any, else the resident with the smallest key is evicted
        (replaced += 1), key = (last-access stamp, admission seq) for LRU and
        (admission seq) for FIFO (reading Q27: ties inside a batch go to the
        earlier admission; a miss may evict one admitted earlier in the same
        batch when the batch has more misses than the capacity).

    Starts empty (SPEC: dynamic policies start with no resident rows).
    State: slot[v] (-1 = absent), owner[s] (-1 = free), stamp[s], seq[s].
    """

    def __init__(self, n: int, capacity: int, policy: int):
        if policy not in (POLICY_FIFO, POLICY_LRU):
            raise ValueError("parameter error: policy must be FIFO or LRU")
        self.C = int(capacity)
        self.policy = policy
        self.slot = np.full(n, -1, dtype=np.int64)
        self.owner = np.full(self.C, -1, dtype=np.int64)
        self.stamp = np.full(self.C, -1, dtype=np.int64)
        self.seq = np.full(self.C, -1, dtype=np.int64)
        self.t = 0
        self.next_seq = 0
        self.hits = self.misses = self.replaced = 0

    def _victim(self) -> int:
        free = np.nonzero(self.owner < 0)[0]
        if free.size:
            return int(free[0])
        if self.policy == POLICY_LRU:
            order = np.lexsort((self.seq, self.stamp))  # primary stamp, then seq
        else:
            order = np.argsort(self.seq, kind="stable")
        return int(order[0])

    def access_batch(self, rows) -> dict:
        rows = [int(v) for v in rows]
        hit = [v for v in rows if self.slot[v] >= 0]
        miss = [v for v in rows if self.slot[v] < 0]
        if self.policy == POLICY_LRU:
            for v in hit:
                self.stamp[self.slot[v]] = self.t
        replaced = 0
        if self.C > 0:
            for v in miss:
                s = self._victim()
                old = int(self.owner[s])
                if old >= 0:
                    self.slot[old] = -1
                    replaced += 1
                self.owner[s] = v
                self.slot[v] = s
                self.stamp[s] = self.t
                self.seq[s] = self.next_seq
                self.next_seq += 1
        self.t += 1
        self.hits += len(hit)
        self.misses += len(miss)
        self.replaced += replaced
        return dict(rows=len(rows), hits=len(hit), misses=len(miss), replaced=replaced)

    def resident(self) -> set:
        return set(int(v) for v in self.owner[self.owner >= 0])
