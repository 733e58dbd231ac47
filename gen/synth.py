"""Seeded synthetic event-log generator (test and bench infrastructure).

This module is shared by the oracle tests and the CUDA path, and holds none of
the method's arithmetic: it never sorts events by case, never forms
directly-follows pairs, never hashes sequences and never counts anything.  It
only draws a log whose *shape* follows the paper's workloads (PAPER.md
Table 1: events / cases / variants / activities) and the recipe
in SURVEY.md §8(d) / DESIGN.md "Input recipe":

* case lengths  : 1 + Poisson(mean - 1), clipped to [1, max_len]; for configs
                  with an exact event count the lengths are nudged by +-1 on
                  hash-chosen cases until the total is exact;
* activities    : a planted variant pool (sequences drawn by a Markov walk on a
                  random activity graph, out-degree 4, Zipf edge weights) split
                  into per-length buckets; each case picks a variant of its own
                  length with Zipf(s=1.1) weights; a fraction of cases instead
                  take a fresh random walk ("random" cases);
* timestamps    : case start ~ U[T0, T0 + 365 d), T0 = 2019-01-01Z in ms; gaps
                  are 0 with probability ``zero_gap_p`` (timestamp ties), else
                  ceil(LogNormal(median 1 h, sigma 1.5)) capped at 7 d;
* row order     : events are shuffled by ascending splitmix64(seed, case, pos),
                  so the ingest order does not depend on how cases are sharded.

Everything per case or per event is a pure function of (seed, global case id,
position), computed with wrapping int64 arithmetic in torch, so the same code
runs on CPU (oracle tests) and on a GPU (bench at 10^8-10^9 events) and yields
bit-identical logs.  The planted ground truth (per-case variant id, pool
sequences) is returned for closed-form pins.
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import torch

T0_MS = 1_546_300_800_000          # 2019-01-01T00:00:00Z
YEAR_MS = 365 * 86_400_000
HOUR_MS = 3_600_000
WEEK_MS = 7 * 86_400_000

# stream ids for the counter-based generator
_S_LEN, _S_FIX, _S_VAR, _S_RND, _S_WALK, _S_START, _S_GAP, _S_ORDER = range(1, 9)

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """Python int (mod 2^64) -> signed int64 value."""
    x &= _M64
    return x - (1 << 64) if x >> 63 else x


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical shift right of an int64 tensor viewed as uint64."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    z = x + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def chash(seed: int, stream: int, a: torch.Tensor, b: torch.Tensor | int = 0) -> torch.Tensor:
    """Counter-based 64-bit hash of (seed, stream, a, b) as int64."""
    k = splitmix64(torch.tensor(_s64(seed * 0x100000001B3 + stream), dtype=torch.int64))
    h = splitmix64(a.to(torch.int64) ^ k.to(a.device))
    bt = torch.as_tensor(b, dtype=torch.int64, device=a.device)
    return splitmix64(h + bt * _GOLDEN)


def _u53(h: torch.Tensor) -> torch.Tensor:
    """Uniform integer in [0, 2^53) from a hash."""
    return _lsr(h, 11)


@dataclass(frozen=True)
class LogSpec:
    name: str
    n_cases: int
    n_activities: int
    mean_len: float
    n_events: int | None      # exact total (None: whatever the lengths sum to)
    pool_size: int            # planted variant pool size
    pool_exact: bool          # every pool variant is used by >= 1 case
    frac_random: float        # fraction of cases drawn as fresh random walks
    max_len: int
    zero_gap_p: float         # probability of a 0 ms gap (timestamp tie)
    seed: int
    # "random": rows fully shuffled, so tied events of a case arrive in random
    # order; "chronological": rows interleaved across cases but each case's
    # events arrive in planted order (ties then keep the planted sequence, so
    # the observed variant count equals the pool size exactly).
    ingest: str = "random"

    def with_(self, **kw) -> "LogSpec":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; shapes from PAPER.md Table 1 (x1 base
# = the _2 row / 2) and SURVEY.md §8(d).
CONFIGS: dict[str, LogSpec] = {
    "tiny": LogSpec("tiny", 1_000, 10, 10.0, None, 20, False, 0.5, 40, 0.02, 1),
    "roadtraffic": LogSpec("roadtraffic", 150_370, 11, 561_470 / 150_370, 561_470,
                           231, True, 0.0, 40, 0.02, 2, "chronological"),
    "bpic2019": LogSpec("bpic2019", 251_734, 42, 1_595_923 / 251_734, 1_595_923,
                        11_973, True, 0.0, 40, 0.02, 3, "chronological"),
    "100M": LogSpec("100M", 10_000_000, 64, 10.0, 100_000_000, 1 << 16, False, 0.0,
                    40, 0.02, 4),
    "1B": LogSpec("1B", 50_000_000, 256, 20.0, 1_000_000_000, 1 << 18, False, 0.0,
                  80, 0.02, 5),
    # long cases (not a BASELINE.json config): the BPIC2018 shape (Table 1:
    # bpic2018_2 = 5,028,532 events / 87,618 cases / 28,457 variants / 41 activities;
    # x1 base = half), mean 57 events per case, fully shuffled rows -- the in-case
    # ranking's O(m) per row and the exact fallback's long cases at their heaviest
    "bpic2018": LogSpec("bpic2018", 43_809, 41, 2_514_266 / 43_809, 2_514_266,
                        28_457, True, 0.0, 400, 0.02, 6),
}


@dataclass
class EventLog:
    """A generated shard: columns in ingest (shuffled) order plus ground truth."""
    case: torch.Tensor        # int64 global case code
    act: torch.Tensor         # int64 activity code
    ts: torch.Tensor          # int64 ms since epoch
    n_activities: int
    n_case_codes: int         # global case dictionary size
    case_lo: int              # this shard's case-code range [case_lo, case_hi)
    case_hi: int
    # planted ground truth (per case of the shard, in case-code order)
    case_len: torch.Tensor
    case_variant: torch.Tensor    # pool index, or -1 for a random walk
    pool_seqs: list               # list of tuples of activity codes

    @property
    def n(self) -> int:
        return int(self.case.numel())

    def act_dtype(self) -> torch.dtype:
        return act_dtype_for(self.n_activities)

    def columns(self, device=None):
        """(case u32-as-int32, act u8/u16-as-int16/u32-as-int32, ts int64) tensors."""
        dev = device or self.case.device
        case = self.case.to(torch.int64).to(torch.int32).to(dev)
        act = self.act.to(self.act_dtype()).to(dev)
        ts = self.ts.to(dev)
        return case, act, ts


def act_dtype_for(n_activities: int) -> torch.dtype:
    if n_activities <= 256:
        return torch.uint8
    if n_activities <= 65536:
        return torch.int16
    return torch.int32


# ---------------------------------------------------------------- host-side pool
def _markov_graph(rng: np.random.Generator, A: int, deg: int = 4):
    d = min(deg, A)
    succ = np.stack([rng.choice(A, size=d, replace=False) for _ in range(A)])
    w = 1.0 / np.arange(1, d + 1) ** 1.1
    w /= w.sum()
    start_perm = rng.permutation(A)
    sw = 1.0 / np.arange(1, A + 1) ** 1.1
    sw /= sw.sum()
    start_w = np.empty(A)
    start_w[start_perm] = sw
    return succ, w, start_w


def _walks(rng, succ, w, start_w, n, length):
    A = succ.shape[0]
    out = np.empty((n, length), dtype=np.int64)
    out[:, 0] = rng.choice(A, size=n, p=start_w)
    for k in range(1, length):
        pick = rng.choice(succ.shape[1], size=n, p=w)
        out[:, k] = succ[out[:, k - 1], pick]
    return out


def _poisson_pmf(lam: float, kmax: int) -> np.ndarray:
    ks = np.arange(kmax + 1)
    logp = -lam + ks * math.log(max(lam, 1e-300)) - np.array([math.lgamma(k + 1) for k in ks])
    p = np.exp(logp) if lam > 0 else (ks == 0).astype(float)
    return p


def _length_pmf(spec: LogSpec) -> np.ndarray:
    """pmf over lengths 1..max_len (index 0 unused)."""
    p = np.zeros(spec.max_len + 1)
    q = _poisson_pmf(spec.mean_len - 1.0, spec.max_len - 1)
    p[1:] = q
    p[spec.max_len] += max(0.0, 1.0 - q.sum())
    return p / p.sum()


def _build_pool(spec: LogSpec, len_counts: np.ndarray):
    """Planted variant pool, bucketed by length.

    Returns (seqs, bucket_start, bucket_size): bucket for length l holds pool ids
    [bucket_start[l], bucket_start[l] + bucket_size[l]).
    """
    rng = np.random.default_rng(spec.seed * 7919 + 17)
    succ, w, start_w = _markov_graph(rng, spec.n_activities)
    A, d = succ.shape
    L = spec.max_len
    pmf = len_counts / max(1, len_counts.sum())
    cap = np.zeros(L + 1, dtype=np.int64)
    for l in range(1, L + 1):
        if len_counts[l] == 0:
            continue
        walks = A * d ** (l - 1) if l < 40 else 1 << 62
        cap[l] = min(int(len_counts[l]) if spec.pool_exact else 1 << 62, walks)
    want = np.zeros(L + 1, dtype=np.int64)
    if spec.pool_exact:           # every occurring length gets >= 1 variant
        want[cap > 0] = 1
    rem = spec.pool_size - int(want.sum())
    order = np.argsort(-pmf, kind="stable")
    while rem > 0:
        room = cap - want
        if room.sum() == 0:
            break
        share = np.minimum(np.floor(rem * pmf).astype(np.int64), room)
        if share.sum() == 0:
            for l in order:
                if rem == 0:
                    break
                if room[l] > 0:
                    want[l] += 1
                    rem -= 1
        else:
            want += share
            rem -= int(share.sum())
    seqs: list = []
    bucket_start = np.zeros(L + 2, dtype=np.int64)
    bucket_size = np.zeros(L + 2, dtype=np.int64)
    for l in range(1, L + 1):
        bucket_start[l] = len(seqs)
        k = int(want[l])
        if k <= 0:
            continue
        got: dict = {}
        tries = 0
        n_walks = A * d ** (l - 1) if l < 40 else 1 << 62
        if 2 * k >= n_walks and n_walks <= 1 << 20:
            allw = np.zeros((n_walks, l), dtype=np.int64)
            idx = np.arange(n_walks)
            allw[:, 0] = idx % A
            rest = idx // A
            for j in range(1, l):
                allw[:, j] = succ[allw[:, j - 1], rest % d]
                rest //= d
            take = np.sort(rng.choice(n_walks, size=k, replace=False))
            for row in map(tuple, allw[take].tolist()):
                got[row] = None
        while len(got) < k:
            batch = _walks(rng, succ, w, start_w, max(64, 2 * (k - len(got))), l)
            for row in map(tuple, batch.tolist()):
                if row not in got:
                    got[row] = None
                    if len(got) == k:
                        break
            tries += 1
            if tries > 200:  # near-exhaustive: enumerate remaining uniformly
                break
        seqs.extend(got.keys())
        bucket_size[l] = len(got)
    return seqs, bucket_start, bucket_size, (succ, w, start_w)


# ---------------------------------------------------------------- per-case draws
def _inv_cdf_table(p: np.ndarray) -> torch.Tensor:
    """Integer inverse-CDF thresholds (in [0, 2^53]) for searchsorted(right=True)."""
    c = np.cumsum(p)
    c = c / c[-1]
    t = np.minimum(np.round(c * float(1 << 53)), float(1 << 53)).astype(np.int64)
    t[-1] = 1 << 53
    return torch.from_numpy(t)


def _gap_table() -> torch.Tensor:
    """65536 quantiles of ceil(LogNormal(median 1 h, sigma 1.5)) ms, capped at 7 d."""
    from statistics import NormalDist
    nd = NormalDist()
    q = (np.arange(65536) + 0.5) / 65536.0
    z = np.array([nd.inv_cdf(float(x)) for x in q])
    g = np.ceil(HOUR_MS * np.exp(1.5 * z))
    g = np.clip(g, 1, WEEK_MS).astype(np.int64)
    return torch.from_numpy(g)


_GAP_TABLE = None


def _gaps() -> torch.Tensor:
    global _GAP_TABLE
    if _GAP_TABLE is None:
        _GAP_TABLE = _gap_table()
    return _GAP_TABLE


def case_lengths(spec: LogSpec, device="cpu") -> torch.Tensor:
    """Per-case length for all global cases (int64[C]), exact total if requested."""
    C = spec.n_cases
    ids = torch.arange(C, dtype=torch.int64, device=device)
    pmf = _length_pmf(spec)
    thr = _inv_cdf_table(pmf[1:]).to(device)
    u = _u53(chash(spec.seed, _S_LEN, ids))
    lens = torch.searchsorted(thr, u, right=True).clamp_(max=spec.max_len - 1) + 1
    if spec.n_events is not None:
        delta = spec.n_events - int(lens.sum())
        prio = chash(spec.seed, _S_FIX, ids)
        order = torch.argsort(prio, stable=True)
        while delta != 0:
            step = 1 if delta > 0 else -1
            ok = (lens[order] < spec.max_len) if step > 0 else (lens[order] > 1)
            cand = order[ok]
            k = min(abs(delta), int(cand.numel()))
            if k == 0:
                raise ValueError("cannot reach the exact event count")
            lens[cand[:k]] += step
            delta -= step * k
    return lens


def generate(spec: LogSpec, case_lo: int = 0, case_hi: int | None = None,
             device="cpu", no_ties: bool = False, shuffle: bool = True) -> EventLog:
    """Draw the shard [case_lo, case_hi) of the log described by ``spec``."""
    C = spec.n_cases
    case_hi = C if case_hi is None else case_hi
    assert 0 <= case_lo <= case_hi <= C
    dev = torch.device(device)
    lens_all = case_lengths(spec, dev)
    len_counts = torch.bincount(lens_all, minlength=spec.max_len + 1).cpu().numpy()
    seqs, bstart, bsize, graph = _build_pool(spec, len_counts)
    succ, w, start_w = graph

    ids_all = torch.arange(C, dtype=torch.int64, device=dev)
    # variant pick: Zipf(1.1) inside the case's length bucket, via one global
    # monotone threshold table (bucket l occupies [l*2^53, (l+1)*2^53)).
    thr_parts, base = [], []
    for l in range(1, spec.max_len + 1):
        k = int(bsize[l])
        if k == 0:
            continue
        zw = 1.0 / np.arange(1, k + 1) ** 1.1
        t = _inv_cdf_table(zw).numpy() + (l << 53)
        thr_parts.append(t)
    thr = torch.from_numpy(np.concatenate(thr_parts)).to(dev) if thr_parts else None
    has_bucket = torch.from_numpy(bsize[: spec.max_len + 1] > 0).to(dev)
    u = _u53(chash(spec.seed, _S_VAR, ids_all))
    variant = torch.full((C,), -1, dtype=torch.int64, device=dev)
    if thr is not None:
        pick = torch.searchsorted(thr, (lens_all << 53) + u, right=True)
        ok = has_bucket[lens_all]
        variant = torch.where(ok, pick, variant)
    if spec.frac_random > 0:
        r = _u53(chash(spec.seed, _S_RND, ids_all))
        rnd = r < int(spec.frac_random * (1 << 53))
        variant = torch.where(rnd, torch.full_like(variant, -1), variant)
    if spec.pool_exact:
        # coverage: the first bsize[l] cases of length l take variants 0..bsize[l]-1
        key = lens_all * C + ids_all
        order = torch.argsort(key, stable=True)
        sl = lens_all[order]
        first = torch.searchsorted(sl, sl, right=False)
        rank = torch.arange(C, device=dev) - first
        bs = torch.from_numpy(bsize[: spec.max_len + 1]).to(dev)
        bst = torch.from_numpy(bstart[: spec.max_len + 1]).to(dev)
        cov = rank < bs[sl]
        variant[order[cov]] = bst[sl[cov]] + rank[cov]

    # ---- slice to the shard
    lens = lens_all[case_lo:case_hi]
    variant = variant[case_lo:case_hi]
    ids = ids_all[case_lo:case_hi]
    n = int(lens.sum())
    case_ev = torch.repeat_interleave(ids, lens)
    off = torch.cumsum(lens, 0) - lens
    pos = torch.arange(n, dtype=torch.int64, device=dev) - torch.repeat_interleave(off, lens)

    # ---- activities
    if seqs:
        flat = torch.tensor([a for s in seqs for a in s], dtype=torch.int64, device=dev)
        soff = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])[:-1]]),
                            dtype=torch.int64, device=dev)
    var_ev = torch.repeat_interleave(variant, lens)
    act = torch.zeros(n, dtype=torch.int64, device=dev)
    pooled = var_ev >= 0
    if seqs and bool(pooled.any()):
        act[pooled] = flat[soff[var_ev[pooled]] + pos[pooled]]
    if bool((~pooled).any()):
        act[~pooled] = _random_walk_acts(spec, case_ev[~pooled], pos[~pooled],
                                         lens, variant, ids, graph, dev)

    # ---- timestamps
    start = T0_MS + torch.remainder(chash(spec.seed, _S_START, ids), YEAR_MS)
    hg = chash(spec.seed, _S_GAP, case_ev, pos)
    gap = _gaps().to(dev)[_lsr(hg, 20) & 0xFFFF]
    if not no_ties and spec.zero_gap_p > 0:
        zero = torch.remainder(hg, 1 << 20) < int(spec.zero_gap_p * (1 << 20))
        gap = torch.where(zero, torch.zeros_like(gap), gap)
    gap = torch.where(pos == 0, torch.zeros_like(gap), gap)
    cs = torch.cumsum(gap, 0)
    ts = torch.repeat_interleave(start, lens) + cs - torch.repeat_interleave(cs[off] if n else cs, lens)

    # ---- ingest order
    if shuffle and n:
        key = chash(spec.seed, _S_ORDER, case_ev, pos)
        if spec.ingest == "chronological":
            # monotone in pos inside a case: base(case) + running sum of
            # positive increments; cases still interleave at random.
            inc = torch.where(pos == 0, _u53(key), (key & ((1 << 45) - 1)) + 1)
            ck = torch.cumsum(inc, 0)
            key = ck - torch.repeat_interleave(ck[off] - inc[off], lens)
        perm = torch.argsort(key, stable=True)
        case_ev, act, ts = case_ev[perm], act[perm], ts[perm]
    return EventLog(case_ev, act, ts, spec.n_activities, C, case_lo, case_hi,
                    lens, variant, seqs)


def _random_walk_acts(spec, case_ev, pos, lens, variant, ids, graph, dev):
    """Fresh Markov walks for the non-pool cases (hash-driven, shard-independent)."""
    succ, w, start_w = graph
    A, d = succ.shape
    rnd_cases = ids[variant < 0]
    rl = lens[variant < 0]
    Lmax = int(rl.max()) if rl.numel() else 0
    st_thr = _inv_cdf_table(start_w).to(dev)
    w_thr = _inv_cdf_table(w).to(dev)
    succ_t = torch.from_numpy(succ).to(dev)
    walk = torch.empty((rnd_cases.numel(), max(Lmax, 1)), dtype=torch.int64, device=dev)
    walk[:, 0] = torch.searchsorted(st_thr, _u53(chash(spec.seed, _S_WALK, rnd_cases, 0)),
                                    right=True).clamp_(max=A - 1)
    for k in range(1, Lmax):
        pk = torch.searchsorted(w_thr, _u53(chash(spec.seed, _S_WALK, rnd_cases, k)),
                                right=True).clamp_(max=d - 1)
        walk[:, k] = succ_t[walk[:, k - 1], pk]
    # map events -> (row in walk, pos)
    row_of_case = torch.full((int(ids.max()) + 1 - int(ids.min()) if ids.numel() else 1,), -1,
                             dtype=torch.int64, device=dev)
    base = int(ids.min()) if ids.numel() else 0
    row_of_case[rnd_cases - base] = torch.arange(rnd_cases.numel(), device=dev)
    return walk[row_of_case[case_ev - base], pos]


def replicate(log: EventLog, k: int) -> EventLog:
    """PAPER.md P:176 methodology: every case duplicated k times under fresh ids.

    Copy j of case c gets code j * n_case_codes + c; rows are concatenated copy
    by copy (ingest order of each copy preserved).
    """
    C = log.n_case_codes
    cases = torch.cat([log.case + j * C for j in range(k)])
    return EventLog(cases, log.act.repeat(k), log.ts.repeat(k), log.n_activities, C * k,
                    0, C * k, log.case_len.repeat(k), log.case_variant.repeat(k), log.pool_seqs)
