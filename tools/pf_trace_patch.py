"""Experiment helper: insert / remove clock64 stamps (PFT) in the tcgen05 prefill kernel for one CTA
(the first compute CTA), written to the trace buffer at [2100 + 16 t + event]. Not part of the build.

  python tools/pf_trace_patch.py apply|revert
"""
import sys
P = "paper_2604_26074_b200/csrc/prefill.cu"
MARK = "  // PFT-TRACE\n"
PTS = [  # (anchor line, event, guard)
    ("        tma_3d(dst + 16384, vm, 0, (int)row, 0, &full[s2]);  // V\n", 0, ""),
    ("        umma_commit(&s_full[t & 1]);\n", 1, ""),
    ("        if (t >= kUStages) mbar_wait(&empty[s2], (uint32_t)((t / kUStages - 1) & 1));\n", 11, ""),
    ("        umma_commit(&pv_done[bb]);  // P(t) consumed; O_bb holds tiles <= t of its parity\n", 2, ""),
    ("      if (lane == 0) mbar_arrive(&vconv[s2]);\n", 3, "lane == 0 && warp == 2"),
    ("      for (int j = 0; j < kTile; ++j) asm volatile(\"\" : \"+r\"(sv_u[j]));  // keep every use after the wait\n", 5, "lane == 0 && q4 == 0"),
    ("      const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])) * p.scale_log2;  // scale > 0\n", 6, "lane == 0 && q4 == 0"),
    ("      if (k > 0) mbar_wait(&pv_done[c], (uint32_t)((k - 1) & 1));\n", 7, "lane == 0 && q4 == 0"),
    ("      tmem_st16(p_c, pw);\n", 8, "lane == 0 && q4 == 0"),
    ("      if (lane == 0) mbar_arrive(&p_full[c]);\n", 9, "lane == 0 && q4 == 0"),
]
PRE = [("      mbar_wait(&s_full[c], (uint32_t)(k & 1));\n", 4, "lane == 0 && q4 == 0"),
       ("        if (t >= kUStages) mbar_wait(&empty[s2], (uint32_t)((t / kUStages - 1) & 1));\n", 10, ""),
       ("      if (t + 2 < nt) issue_s(t + 2);  // first: softmax(t + 2) waits for it\n", 12, "leader"),
       ("      mbar_wait(&p_full[bb], (uint32_t)((t >> 1) & 1));\n", 13, "leader")]
DEF = ('#define PFT(ev, tt) do { if (p.trace && cta == 0 && (tt) < 64) { long long c_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)); '
       'p.trace[2100 + (tt) * 16 + (ev)] = (unsigned long long)c_; } } while (0)\n')
s = open(P).read()
if sys.argv[1] == "apply":
    assert MARK not in s
    s = s.replace("constexpr int kUThreads = 14 * 32;", DEF + "constexpr int kUThreads = 14 * 32;", 1)
    for a, ev, g in PTS:
        assert s.count(a) == 1, a
        st = f"PFT({ev}, t);" if not g else f"if ({g}) PFT({ev}, t);"
        s = s.replace(a, a + " " * (len(a) - len(a.lstrip())) + st + MARK.strip() + "\n")
    for a, ev, g in PRE:
        assert s.count(a) == 1, a
        st = f"PFT({ev}, t);" if not g else f"if ({g}) PFT({ev}, t);"
        s = s.replace(a, " " * (len(a) - len(a.lstrip())) + st + MARK.strip() + "\n" + a)
else:
    s = "".join(l for l in s.splitlines(True) if "// PFT-TRACE" not in l and not l.startswith("#define PFT("))
open(P, "w").write(s)
