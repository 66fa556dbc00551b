"""TEST INFRASTRUCTURE ONLY -- the paper's algorithms written out step by step, in its order and notation.

Pure Python, for tiny instances.  Used to pin the oracle: Theorem 1 makes
"BF, IIB and IIIB return the same neighbour lists" a checkable invariant, and the cost models
(Eq. 2-4) become exact counter laws.

* ``block_nested_loops_join``  -- Alg. 1: R blocks outer, S blocks inner, pruneScore
                                   initialised to 0 per R block (line 3), OutputKNN after the inner loop.
* ``kernel_bf``                -- Alg. 2.
* ``kernel_iib``               -- Alg. 3.
* ``kernel_iiib``              -- Alg. 4 with MinPruneScore.
* ``CandidateSet``             -- the KNN candidate set with pruneScore.

Readings: c1 ties to the lower S id -- the strict ``v > pruneScore`` test of Alg. 2 line 5
with S visited in ascending id order, evicting the highest id among tied minima, yields exactly that;
c2 zero scores never admitted; c3 pruneScore = 0 while under-full; c4 the accumulator A is visited in
ascending S id; c9 strict index trigger ``t > MinPruneScore``; c10 frequency order count desc then
dimension asc, absent dimensions last.
"""
from __future__ import annotations

from dataclasses import dataclass, field


def rows_of(csr):
    """HostCSR -> list of rows, each a list of (d, w) pairs ascending in d."""
    out = []
    for i in range(csr.n_rows):
        idx, val = csr.row(i)
        if val is None:
            out.append([(int(d), 1) for d in idx])
        elif val.dtype.kind == "i":
            out.append([(int(d), int(w)) for d, w in zip(idx, val)])
        else:
            out.append([(int(d), float(w)) for d, w in zip(idx, val)])
    return out


@dataclass
class Counters:
    """SPEC.md:133-136 CostCounters, Eq. 2-4."""
    feature_visits: int = 0      # BF: |r|+|s| charged per pair (Eq. 3)
    feature_advances: int = 0    # BF: true merge iterator advances (<= |r|+|s|, Eq. 2)
    postings_built: int = 0      # Eq. 4 first term
    postings_visited: int = 0    # Eq. 4 second term
    residual_visits: int = 0     # Alg. 4 line 21 merge advances
    r_blocks_read: int = 0
    s_blocks_read: int = 0


def dot(r, s, counters: Counters | None = None):
    """Alg. 2 lines 8-23: the two-iterator merge."""
    ret = 0
    i = j = 0
    adv = 0
    while i < len(r) and j < len(s):
        fr, fs = r[i], s[j]
        if fr[0] == fs[0]:
            ret = ret + fr[1] * fs[1]
            i += 1
            j += 1
            adv += 2
        elif fr[0] > fs[0]:
            j += 1
            adv += 1
        else:
            i += 1
            adv += 1
    if counters is not None:
        counters.feature_advances += adv
    return ret


@dataclass
class CandidateSet:
    """bounded top-k with pruneScore(r) = score of the k-th neighbour (0 while
    under-full)."""
    k: int
    entries: list = field(default_factory=list)   # (score, s_id)

    @property
    def prune_score(self):
        return min(e[0] for e in self.entries) if len(self.entries) == self.k else 0

    def offer(self, s_id, v) -> bool:
        """Alg. 2 lines 5-7: if v > pruneScore(r) insert s and update pruneScore."""
        if not (v > self.prune_score):
            return False
        if len(self.entries) == self.k:
            # evict the minimum; among tied minima the highest id (reading c4)
            worst = min(self.entries, key=lambda e: (e[0], -e[1]))
            self.entries.remove(worst)
        self.entries.append((v, s_id))
        return True

    def output(self):
        """OutputKNN (Alg. 1 line 7): score desc, id asc."""
        return sorted(self.entries, key=lambda e: (-e[0], e[1]))


def kernel_bf(Br, Bs, cands, counters: Counters, **_):
    """Alg. 2: every pair, dot(), strict threshold insert."""
    for ri, r in Br:
        for si, s in Bs:
            counters.feature_visits += len(r) + len(s)   # Eq. 3 charge
            v = dot(r, s, counters)
            if v > cands[ri].prune_score:
                cands[ri].offer(si, v)


def create_inverted_list_iib(Bs, counters: Counters):
    """Alg. 3 lines 5-8: insert (s, s[d]) into I_d for every feature of every s."""
    inv = {}
    for si, s in Bs:
        for d, w in s:
            inv.setdefault(d, []).append((si, w))
            counters.postings_built += 1
    return inv


def find_matches_iib(ri, r, inv, cands, counters: Counters):
    """Alg. 3 lines 9-17."""
    A = {}
    for d, rd in r:
        for si, sd in inv.get(d, ()):
            A[si] = A.get(si, 0) + rd * sd
            counters.postings_visited += 1
    for si in sorted(A):                     # reading c4: ascending S id
        if A[si] != 0 and A[si] > cands[ri].prune_score:
            cands[ri].offer(si, A[si])
    return A


def kernel_iib(Br, Bs, cands, counters: Counters, **_):
    inv = create_inverted_list_iib(Bs, counters)
    for ri, r in Br:
        find_matches_iib(ri, r, inv, cands, counters)


def frequency_profile(Br, D):
    """Alg. 4 lines 6-7: dimension order by non-zero count in B_r (desc, then dimension asc; dimensions
    absent from B_r last, ascending -- reading c10) and maxWeight_d(B_r)."""
    count, maxw = {}, {}
    for _, r in Br:
        for d, w in r:
            count[d] = count.get(d, 0) + 1
            maxw[d] = max(maxw.get(d, 0), w)
    present = sorted(count, key=lambda d: (-count[d], d))
    rank = {d: i for i, d in enumerate(present)}
    n = len(present)
    order_key = lambda d: rank[d] if d in rank else n + d
    return order_key, maxw


def create_inverted_list_iiib(Bs, Br, min_prune, D, counters: Counters):
    """Alg. 4 lines 5-14: features of s in profile order; t += maxWeight_d(B_r)*w; once t > MinPruneScore
    insert (s, w) into I_d and remove the feature from s.  Returns (I, residual s' per s)."""
    order_key, maxw = frequency_profile(Br, D)
    inv, residual = {}, {}
    for si, s in Bs:
        t = 0
        res = []
        for d, w in sorted(s, key=lambda f: order_key(f[0])):
            t = t + maxw.get(d, 0) * w
            if t > min_prune:
                inv.setdefault(d, []).append((si, w))
                counters.postings_built += 1
            else:
                res.append((d, w))
        residual[si] = sorted(res)           # "Remove feature" as flags; s' stays d-sorted
    return inv, residual


def find_matches_iiib(ri, r, inv, residual, cands, counters: Counters):
    """Alg. 4 lines 15-24: accumulate over indexed postings, then complete with dot(r, s') (line 21)."""
    A = {}
    for d, rd in r:
        for si, sd in inv.get(d, ()):
            A[si] = A.get(si, 0) + rd * sd
            counters.postings_visited += 1
    for si in sorted(A):
        if A[si] == 0:
            continue
        c = Counters()
        A[si] = A[si] + dot(r, residual[si], c)
        counters.residual_visits += c.feature_advances
        if A[si] > cands[ri].prune_score:
            cands[ri].offer(si, A[si])
    return A


def kernel_iiib(Br, Bs, cands, counters: Counters, D=None, **_):
    min_prune = min_prune_score([cands[ri] for ri, _ in Br])
    inv, residual = create_inverted_list_iiib(Bs, Br, min_prune, D, counters)
    for ri, r in Br:
        find_matches_iiib(ri, r, inv, residual, cands, counters)


def min_prune_score(sets):
    """MinPruneScore = min over r in B_r of pruneScore(r) (0 when any set is under-full)."""
    return min((c.prune_score for c in sets), default=0)


KERNELS = {"bf": kernel_bf, "iib": kernel_iib, "iiib": kernel_iiib}


def block_nested_loops_join(R_rows, S_rows, k, kernel="iib", r_block=None, s_block=None, D=None):
    """Alg. 1.  Blocks are contiguous row ranges of r_block / s_block vectors (the
    disk-page budget of §4.1 is out of scope; only the loop structure matters here).
    Returns (list of per-r [(s_id, score), ...] in rank order, Counters)."""
    counters = Counters()
    kern = KERNELS[kernel]
    nr, ns = len(R_rows), len(S_rows)
    r_block = r_block or max(nr, 1)
    s_block = s_block or max(ns, 1)
    out = [None] * nr
    for r0 in range(0, nr, r_block):                                  # line 1
        Br = [(i, R_rows[i]) for i in range(r0, min(nr, r0 + r_block))]   # line 2 ReadBlock
        counters.r_blocks_read += 1
        cands = {i: CandidateSet(k) for i, _ in Br}                   # line 3 InitPruneScore
        for s0 in range(0, ns, s_block):                              # line 4
            Bs = [(j, S_rows[j]) for j in range(s0, min(ns, s0 + s_block))]  # line 5
            counters.s_blocks_read += 1
            kern(Br, Bs, cands, counters, D=D)                        # line 6
        for i, _ in Br:                                               # line 7 OutputKNN
            out[i] = [(s, v) for v, s in cands[i].output()]
    return out, counters
