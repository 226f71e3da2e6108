"""DAK CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the DAK decode hot path computes,
written from the paper (/root/reference/PAPER.md, arxiv 2604.26074; cited as P:L<line>) and,
for interfaces only, from SPEC.md (cited as S:L<line>).

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
    ``--impl reference`` legs may import anything from this package. The product path
    (``paper_2604_26074_b200``) never imports it and shares no code with it.
  * Floating point is float64 (or exact ``fractions.Fraction``) unless a function says otherwise.
  * Every function cites the passage it follows. Where the paper is silent or garbled, the
    reading taken is listed in DESIGN.md "Readings" (R1..R14 of SURVEY.md §8(c)).

Modules:
  planner   — effective bandwidth, turning points, three-phase greedy (exact + unit/double),
              uniform baseline, LP-vertex brute force, closed-form optimum, capacity -> R.
  partition — tile-row partition, SM/CTA role assignment (paper rule + B200 row-range rule),
              multicast clusters, host traffic / read amplification (Table 1).
  kernels   — bf16 decode, split GEMV / skinny GEMM, split paged GQA decode attention,
              split-KV partial + LSE merge.
  models    — OPT-30B / Llama-3-70B operator lists and footprints.
"""
