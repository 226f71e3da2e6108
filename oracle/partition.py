"""Partition / scheduling oracle (TEST INFRASTRUCTURE).

Paper passages followed:
  * A (weights or KV) is split along M into m x K tile rows; tile row 0 is in
    host memory, the rest in GPU memory (reading R7: host = the LEADING rows).
  * each SM reads exactly one tier; the number of host SMs is set by the target
    ratio, execution-wave alignment and the congestion cap.
  * Table 1: without multicast a host tile consumed by several SMs crosses the
    link once per consumer (read amplification); P:L562-564 — with TMA multicast the tile is
    fetched once per cluster of consumers.
  * attention KV partitioned along the batch dimension (paper mode).

Interfaces follow SPEC.md partitioner. The B200 row-range rule is the design's own
("CTA roles"), pinned here as plain integer arithmetic.
"""
from __future__ import annotations

import math
from fractions import Fraction


def round_half_up(v) -> int:
    """floor(v + 1/2) in exact arithmetic."""
    return math.floor(Fraction(v) + Fraction(1, 2))


def partition_op(M: int, tile_m: int, x) -> tuple[int, int]:
    """(host tile rows, GPU tile rows) for ratio x: host = round_half_up(x * ceil(M/tile_m))."""
    if tile_m <= 0 or M <= 0:
        raise ValueError("dims must be positive")
    if tile_m > M:
        raise ValueError("tile_m > M")
    rows = -(-M // tile_m)
    host = round_half_up(Fraction(x) * rows)
    host = min(max(host, 0), rows)
    return host, rows - host


def wave_aligned_sms(host_rows: int, share: int) -> int:
    """Paper wave alignment, reading R9:
    the largest n <= share such that host_rows mod n == 0 AND ceil(host_rows/n) ==
    ceil(host_rows/share) (tiles divide evenly without adding a wave — S:L292's example and
    S:L320's "never increases waves" invariant, which S:L289/S:L325's "largest divisor" alone
    would violate, e.g. 8 rows / share 3); if no such n exists, keep the share."""
    if host_rows <= 0:
        return 0
    share = max(1, share)
    waves = -(-host_rows // share)
    for n in range(share, 0, -1):
        if host_rows % n == 0 and -(-host_rows // n) == waves:
            return n
    return share


def assign_sms(host_rows: int, gpu_rows: int, sm_count: int, cap: int | None = None) -> tuple[int, int]:
    """Paper SM role assignment.

    proportional share = floor(sm_count * host_rows / total_rows), at least 1 when host rows exist
    and at most sm_count - 1 when GPU rows exist; with congestion control the share is capped
    at `cap` before wave alignment. Returns (n_sm_host, n_sm_gpu).
    """
    total = host_rows + gpu_rows
    if host_rows == 0:
        return 0, sm_count
    if sm_count < 2 and gpu_rows > 0:
        raise ValueError("need at least one SM per tier")
    share = (sm_count * host_rows) // total
    share = max(1, share)
    if gpu_rows > 0:
        share = min(share, sm_count - 1)
    if cap is not None:
        share = min(share, cap)
    n_host = wave_aligned_sms(host_rows, share)
    return n_host, sm_count - n_host


def consumers_per_host_row(N: int, tile_n: int) -> int:
    """Output column blocks that consume every host tile row of a dense GEMM: ceil(N/tile_n) (Table 1)."""
    return -(-N // tile_n)


def fetches_per_row(consumers: int, multicast: bool, cluster_max: int) -> int:
    """Link fetches of one host tile row: one per consumer without multicast, one per cluster with it."""
    if not multicast:
        return consumers
    return -(-consumers // max(1, cluster_max))


def host_traffic(host_bytes: int, N: int, tile_n: int, multicast: bool = False, cluster_max: int = 1) -> int:
    """Bytes crossing the host link for one GEMM over a host block (Table 1)."""
    return host_bytes * fetches_per_row(consumers_per_host_row(N, tile_n), multicast, cluster_max)


# ----------------------------------------------------------------------------------------------
# B200 design rules — pure integer arithmetic, pinned bit-exactly against the ABI
# ----------------------------------------------------------------------------------------------


def balanced_ranges(R: int, n: int) -> list[tuple[int, int]]:
    """Split R rows over n CTAs into contiguous ranges [floor(jR/n), floor((j+1)R/n)):
    sizes differ by at most one row — row-granular wave alignment."""
    if n <= 0:
        return []
    return [((j * R) // n, ((j + 1) * R) // n) for j in range(n)]


def linear_row_ranges(M: int, h: int, n_cta_host: int, n_cta_hbm: int):
    """Row ownership for dak_linear: host CTAs split rows [0,h), HBM CTAs split [h,M)."""
    out = []
    for a, b in balanced_ranges(h, n_cta_host):
        out.append(("host", a, b))
    for a, b in balanced_ranges(M - h, n_cta_hbm):
        out.append(("hbm", h + a, h + b))
    return out


def host_pages_prefix(n_pages: int, ratio, chunk_pages: int) -> int:
    """Attention page placement (reading in DESIGN.md): the oldest
    round_half_up(ratio * n_chunks) split-KV chunks of a sequence live on the host."""
    n_chunks = -(-n_pages // chunk_pages)
    host_chunks = round_half_up(Fraction(ratio) * n_chunks)
    return min(n_pages, host_chunks * chunk_pages)


def batch_split_host_requests(B: int, ratio) -> int:
    """Paper attention mode: whole requests on host; round_half_up(ratio * B) of them."""
    return min(B, max(0, round_half_up(Fraction(ratio) * B)))


def kv_place_chunk_major(seq_lens, page_size: int, max_pages: int, chunk_pages: int, host_units: int):
    """KV placement of one attention op (reading R15 of DESIGN.md; "tile row 0 in host
    memory"): the op's host units are its OLDEST split-KV chunks, taken chunk-major --
    chunk 0 of request 0, 1, ..., B-1, then chunk 1 of every request that has one, ... Host pages
    are numbered 0, 1, ... in (request, page) order, every other block-table entry (HBM, including
    the max_pages - filled entries later decode tokens use) likewise; a host entry carries bit 31.

    Written as the enumeration it describes. Returns (block table [B][max_pages] of uint32,
    host pages, HBM pages, host tokens)."""
    B = len(seq_lens)
    filled = [-(-int(L) // page_size) for L in seq_lens]
    if any(f > max_pages for f in filled):
        raise ValueError("seq_len beyond max_pages")
    chunks = [-(-f // chunk_pages) for f in filled]
    order = []  # (request, chunk) units, oldest first, chunk-major
    for c in range(max(chunks) if chunks else 0):
        for b in range(B):
            if c < chunks[b]:
                order.append((b, c))
    if host_units > len(order):
        raise ValueError("more host units than chunks")
    host_chunks = [0] * B
    for b, c in order[:host_units]:
        host_chunks[b] += 1
    table = [[0] * max_pages for _ in range(B)]
    ih = ig = host_tokens = 0
    for b in range(B):
        hp = min(host_chunks[b] * chunk_pages, filled[b])
        for p in range(max_pages):
            if p < hp:
                table[b][p] = ih | 0x80000000
                ih += 1
            else:
                table[b][p] = ig
                ig += 1
        host_tokens += min(hp * page_size, int(seq_lens[b]))
    return table, ih, ig, host_tokens


def calib_choice(table, n_host, window, tolerance: float):
    """Congestion-control operating point from the calibration sweep (reading R24 of
    DESIGN.md): table[i][j] = (HBM B/s, host B/s) of a split op run end to end at the balanced ratio
    r* with n_host[i] host CTAs and window[j] requests in flight per host CTA (bytes of each tier /
    the op's time). Its aggregate HBM + host (summed in that order, IEEE double) is the op's
    end-to-end throughput ("the exact SM allocation to the host that maximizes end-to-end
    throughput"); among the points within `tolerance` of the best -- aggregate >=
    best * (1 - tolerance) -- the fewest host CTAs, then the smallest window ("provisions exactly
    enough SMs ... and avoid congestion"); ties: the first index. Returns (i, j)."""
    agg = [[float(table[i][j][0]) + float(table[i][j][1]) for j in range(len(window))] for i in range(len(n_host))]
    best = max(max(row) for row in agg)
    thr = best * (1.0 - tolerance)
    cands = [(n_host[i], window[j], i, j) for i in range(len(n_host)) for j in range(len(window)) if agg[i][j] >= thr]
    n_min = min(c[0] for c in cands)
    w_min = min(c[1] for c in cands if c[0] == n_min)
    return next((c[2], c[3]) for c in cands if c[0] == n_min and c[1] == w_min)


def kv_host_units_keep_ratio(h0: int, n0: int, n_new: int) -> int:
    """Host units of an attention op whose chunk count grew from n0 to n_new while it keeps the
    planner's ratio x = h0 / n0 (P:L466 per-op ratio x_i; reading R23): round-half-up(x * n_new), the
    unit rounding of reading R6, in exact rationals, at most n_new."""
    if n0 == 0:
        return 0
    return min(n_new, round_half_up(Fraction(h0, n0) * n_new))


def kv_replace(old_table, seq_lens, page_size: int, max_pages: int, chunk_pages: int, host_units: int,
               host_pool_pages: int, hbm_pool_pages: int):
    """KV placement across decode steps (reading R23 of DESIGN.md). As the
    requests grow, the planner is re-run for the new context and the attention op gets new host
    units; the tier of every block-table entry is then the chunk-major placement of
    kv_place_chunk_major for the NEW lengths and host units (P:L321-323 oldest rows on the host).
    A page keeps its pool slot when its tier does not change; a page whose tier changes takes the
    lowest slot of the destination pool that the OLD table does not reference (slots freed by this
    re-placement are reused only by the next one, so every copy reads a slot nobody writes).

    Written as the enumeration it describes. Returns (new table [B][max_pages] of uint32, moves as
    (request, page, old entry, new entry) in (request, page) order). Raises ValueError when a pool
    runs out of free slots."""
    HOST = 0x80000000
    fresh, _, _, _ = kv_place_chunk_major(seq_lens, page_size, max_pages, chunk_pages, host_units)
    B = len(seq_lens)
    used_h = set()
    used_g = set()
    for b in range(B):
        for p in range(max_pages):
            e = int(old_table[b][p])
            if e & HOST:
                used_h.add(e & 0x7FFFFFFF)
            else:
                used_g.add(e)
    free_h = [i for i in range(host_pool_pages) if i not in used_h]
    free_g = [i for i in range(hbm_pool_pages) if i not in used_g]
    new = [[0] * max_pages for _ in range(B)]
    moves = []
    for b in range(B):
        for p in range(max_pages):
            old = int(old_table[b][p])
            want_host = bool(fresh[b][p] & HOST)
            if bool(old & HOST) == want_host:
                new[b][p] = old
                continue
            pool = free_h if want_host else free_g
            if not pool:
                raise ValueError("no free slot in the destination pool")
            slot = pool.pop(0)
            new[b][p] = (slot | HOST) if want_host else slot
            moves.append((b, p, old, new[b][p]))
    return new, moves


def linear_splitk_items(M: int, h: int, splits: int, block: int = 128):
    """Row ownership of a split-K dak_linear launch: every tier is cut into blocks
    of `block` rows (the last may be short) and every block into `splits` K ranges; CTA j of a tier
    takes K split j % splits of block j // splits. Host CTAs first (rows [0, h)), then HBM (rows
    [h, M)). Returns [(tier, row_begin, row_end)] per CTA."""
    out = []
    for tier, lo, hi in (("host", 0, h), ("hbm", h, M)):
        n_blocks = -(-(hi - lo) // block)
        for j in range(n_blocks * splits):
            b = j // splits
            out.append((tier, lo + b * block, min(hi, lo + (b + 1) * block)))
    return out
