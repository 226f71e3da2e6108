"""Thin ctypes binding of libdak.so (include/dak.h). Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts Python
values / torch tensors (device memory and streams are torch plumbing) to the C ABI and raises
``DakError`` on a non-OK status. There is no fallback: if libdak.so is missing, importing this
module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libdak.so")

OK, EINVAL, ECAPACITY, EUNSUPPORTED, ECUDA, ENCCL = 0, 1, 2, 3, 4, 5
STATUS = {0: "OK", 1: "EINVAL", 2: "ECAPACITY", 3: "EUNSUPPORTED", 4: "ECUDA", 5: "ENCCL"}
OP_LINEAR, OP_ATTENTION = 0, 1
PLAN_EXACT, PLAN_BALANCED = 0, 1
ACT_NONE, ACT_RELU = 0, 1
HOST_BIT = 0x80000000


class DakError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS.get(status, str(status))


if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libdak.so not built at {_LIB_PATH}; run `python -m paper_2604_26074_b200.build`")
lib = C.CDLL(_LIB_PATH)


# ------------------------------------------------------------------------------------- structs
class dak_hw(C.Structure):
    _fields_ = [("hbm_bps", C.c_double), ("link_bps", C.c_double), ("host_dram_bps", C.c_double),
                ("host_capacity_bytes", C.c_int64), ("host_latency_s", C.c_double)]


class dak_op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("n_units", C.c_int64), ("unit_bytes", C.c_int64),
                ("total_bytes", C.c_int64), ("t_comp_s", C.c_double)]


class dak_op_plan(C.Structure):
    _fields_ = [("host_units", C.c_int64), ("host_bytes", C.c_int64), ("ratio", C.c_double), ("phase", C.c_int32),
                ("reserved", C.c_int32), ("latency_s", C.c_double)]


class dak_launch_cfg(C.Structure):
    _fields_ = [("n_cta_host", C.c_int32), ("n_cta_hbm", C.c_int32), ("window", C.c_int32), ("stages", C.c_int32),
                ("congestion_control", C.c_int32), ("pdl", C.c_int32), ("force_path", C.c_int32),
                ("l2_policy", C.c_int32), ("cluster", C.c_int32), ("host_inflight_kb", C.c_int32)]


class dak_linear_args(C.Structure):
    _fields_ = [("w_host", C.c_void_p), ("w_hbm", C.c_void_p), ("M", C.c_int64), ("K", C.c_int64), ("h", C.c_int64),
                ("kc", C.c_int32), ("N", C.c_int32), ("x", C.c_void_p), ("y", C.c_void_p), ("bias", C.c_void_p),
                ("residual", C.c_void_p), ("act", C.c_int32), ("reserved", C.c_int32), ("cfg", dak_launch_cfg),
                ("ldy", C.c_int64), ("l2_prefetch", C.c_void_p), ("l2_prefetch_bytes", C.c_int64),
                ("ln_w", C.c_void_p), ("ln_b", C.c_void_p), ("ln_stats", C.c_void_p), ("ln_parts", C.c_int32),
                ("ln_rms", C.c_int32), ("ln_eps", C.c_float), ("reserved2", C.c_int32), ("stats_out", C.c_void_p),
                ("x_swiglu", C.c_int32), ("reserved3", C.c_int32), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_int64)]


class dak_linear_launch_info(C.Structure):
    _fields_ = [("grid", C.c_int32), ("n_cta_host", C.c_int32), ("n_cta_hbm", C.c_int32), ("threads", C.c_int32),
                ("stages_hbm", C.c_int32), ("window_host", C.c_int32), ("smem_bytes", C.c_int32), ("path", C.c_int32),
                ("rows_per_cta_host_max", C.c_int64), ("rows_per_cta_hbm_max", C.c_int64),
                ("hbm_bytes", C.c_int64), ("host_bytes", C.c_int64), ("cluster", C.c_int32), ("ksplit", C.c_int32),
                ("host_gate", C.c_int32), ("kblock", C.c_int32)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("dak_last_error", C.c_char_p, [])
_sig("dak_version", C.c_char_p, [])
_sig("dak_device_sms", C.c_int32, [C.POINTER(C.c_int32)])
_sig("dak_trace_enable", C.c_int32, [C.c_void_p, C.c_int32])
_sig("dak_trace_count", C.c_int32, [])
_sig("dak_trace_launch", C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int32)])
_sig("dak_plan_ratios", C.c_int32, [C.POINTER(dak_hw), C.POINTER(dak_op), C.c_int32, C.c_int64, C.c_int32,
                                    C.POINTER(dak_op_plan), C.POINTER(C.c_double)])
_sig("dak_host_alloc", C.c_int32, [C.c_size_t, C.c_int32, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)])
_sig("dak_host_free", C.c_int32, [C.c_void_p])
_sig("dak_linear_packed_bytes", C.c_size_t, [C.c_int64, C.c_int64, C.c_int32])
_sig("dak_pack_linear", C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p])
_sig("dak_linear_default_kc", C.c_int32, [C.c_int64, C.c_int64, C.c_int32])
_sig("dak_linear_query", C.c_int32, [C.POINTER(dak_linear_args), C.POINTER(dak_linear_launch_info)])
_sig("dak_linear_cta_rows", C.c_int32, [C.POINTER(dak_linear_args), C.c_int32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
_sig("dak_linear", C.c_int32, [C.POINTER(dak_linear_args), C.c_void_p])
_sig("dak_linear_workspace_size", C.c_size_t, [C.POINTER(dak_linear_args)])

class dak_attention_args(C.Structure):
    _fields_ = [("q", C.c_void_p), ("out", C.c_void_p), ("k_hbm", C.c_void_p), ("v_hbm", C.c_void_p),
                ("k_host", C.c_void_p), ("v_host", C.c_void_p), ("block_table", C.c_void_p), ("seq_lens", C.c_void_p),
                ("B", C.c_int32), ("Hq", C.c_int32), ("Hkv", C.c_int32), ("d", C.c_int32), ("page_size", C.c_int32),
                ("max_pages", C.c_int32), ("chunk_pages", C.c_int32), ("scale", C.c_float), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("cfg", dak_launch_cfg), ("q_row_stride", C.c_int64),
                ("k_new", C.c_void_p), ("v_new", C.c_void_p), ("kv_new_stride", C.c_int64)]


_sig("dak_pack_kv_pages", C.c_int32, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p])
_sig("dak_attention_workspace_size", C.c_int32, [C.POINTER(dak_attention_args), C.POINTER(C.c_size_t)])
_sig("dak_attention", C.c_int32, [C.POINTER(dak_attention_args), C.c_void_p])
_sig("dak_kv_append", C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_void_p])

EXPORTED = ["dak_pack_kv_pages", "dak_attention_workspace_size", "dak_attention", "dak_kv_append",
            "dak_last_error", "dak_version", "dak_device_sms", "dak_plan_ratios", "dak_host_alloc", "dak_host_free",
            "dak_linear_packed_bytes", "dak_pack_linear", "dak_linear_default_kc", "dak_linear_query",
            "dak_linear_cta_rows", "dak_linear", "dak_linear_workspace_size", "dak_trace_enable", "dak_trace_count", "dak_trace_launch"]


def _check(st: int):
    if st != OK:
        raise DakError(st, (lib.dak_last_error() or b"").decode())


def _ptr(t) -> int | None:
    """Tensor / int / None -> raw address."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(s) -> int | None:
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def version() -> str:
    return lib.dak_version().decode()


TRACE_KINDS = {1: "linear", 2: "attention", 3: "combine", 4: "append", 5: "layernorm", 6: "embed", 7: "splitk_reduce", 8: "prefill",
               9: "residual_norm", 10: "silu_mul"}


def trace_enable(dev_buf, max_launches: int):
    """Record per-CTA globaltimer stamps of the next max_launches per-op launches (dak.h)."""
    _check(lib.dak_trace_enable(_ptr(dev_buf), int(max_launches)))


def trace_launches() -> list:
    out = []
    for i in range(lib.dak_trace_count()):
        k, g = C.c_int32(), C.c_int32()
        a, b = C.c_int64(), C.c_int64()
        _check(lib.dak_trace_launch(i, C.byref(k), C.byref(a), C.byref(b), C.byref(g)))
        out.append(dict(kind=TRACE_KINDS.get(k.value, k.value), a=a.value, b=b.value, grid=g.value))
    return out


def device_sms() -> int:
    v = C.c_int32()
    _check(lib.dak_device_sms(C.byref(v)))
    return v.value


# ------------------------------------------------------------------------------------- planner
def plan_ratios(hw: dict, ops: list, y_req_bytes: int, mode: int = PLAN_EXACT):
    """dak_plan_ratios: hw = {hbm_bps, link_bps, host_dram_bps, host_capacity_bytes};
    ops = [{kind, n_units, unit_bytes, total_bytes, T}]. Returns (list of plan dicts, objective)."""
    h = dak_hw(float(hw["hbm_bps"]), float(hw["link_bps"]), float(hw.get("host_dram_bps", hw["link_bps"])),
               int(hw.get("host_capacity_bytes", -1)), float(hw.get("host_latency_s", 0.0)))
    n = len(ops)
    arr = (dak_op * max(n, 1))()
    for i, o in enumerate(ops):
        k = o.get("kind", OP_LINEAR)
        arr[i].kind = {"linear": OP_LINEAR, "attention": OP_ATTENTION}.get(k, k) if isinstance(k, str) else int(k)
        arr[i].n_units = int(o["n_units"])
        arr[i].unit_bytes = int(o["unit_bytes"])
        arr[i].total_bytes = int(o["total_bytes"])
        arr[i].t_comp_s = float(o["T"])
    out = (dak_op_plan * max(n, 1))()
    obj = C.c_double()
    _check(lib.dak_plan_ratios(C.byref(h), arr, n, int(y_req_bytes), int(mode), out, C.byref(obj)))
    res = [dict(host_units=out[i].host_units, host_bytes=out[i].host_bytes, ratio=out[i].ratio,
                phase=out[i].phase, latency=out[i].latency_s) for i in range(n)]
    return res, obj.value


# ------------------------------------------------------------------------------------- planner inputs, placement
class dak_model(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
                ("tp_size", C.c_int32), ("fused_qkv", C.c_int32), ("fused_gate_up", C.c_int32),
                ("include_head", C.c_int32)]


class dak_op_desc(C.Structure):
    _fields_ = [("layer", C.c_int32), ("role", C.c_int32), ("M", C.c_int64), ("K", C.c_int64), ("flops", C.c_double)]


ROLES = {0: "q", 1: "k", 2: "v", 3: "qkv", 4: "o", 5: "up", 6: "down", 7: "gate", 8: "gate_up", 9: "attn", 10: "head"}

_sig("dak_global_offload_bytes", C.c_int32, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                             C.POINTER(C.c_double)])
_sig("dak_decode_ops", C.c_int32, [C.POINTER(dak_model), C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                   C.c_double, C.POINTER(dak_op), C.POINTER(dak_op_desc), C.c_int32,
                                   C.POINTER(C.c_int32)])
_sig("dak_kv_place", C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int64)])
_sig("dak_kv_replace", C.c_int32, [C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                   C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)])
_sig("dak_kv_migrate", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p])
EXPORTED += ["dak_global_offload_bytes", "dak_decode_ops", "dak_kv_place", "dak_kv_replace", "dak_kv_migrate"]


def global_offload_bytes(weight_bytes: int, kv_bytes: int, hbm_budget_bytes: int, host_capacity_bytes: int = -1):
    """dak_global_offload_bytes -> (y_req bytes, R)."""
    y, r = C.c_int64(), C.c_double()
    _check(lib.dak_global_offload_bytes(int(weight_bytes), int(kv_bytes), int(hbm_budget_bytes),
                                        int(host_capacity_bytes), C.byref(y), C.byref(r)))
    return y.value, r.value


def model(family: int, n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, tp_size=1, fused_qkv=1,
          fused_gate_up=1, include_head=1) -> dak_model:
    return dak_model(int(family), int(n_layers), int(hidden), int(n_heads), int(n_kv_heads), int(head_dim), int(ffn),
                     int(vocab), int(tp_size), int(fused_qkv), int(fused_gate_up), int(include_head))


def decode_ops(m: dak_model, batch: int, context: int, unit_rows: int, chunk_tokens: int, peak_linear: float,
               peak_attn: float) -> list:
    """dak_decode_ops -> list of dicts (kind, n_units, unit_bytes, total_bytes, T, layer, role, M, K, flops)."""
    n = C.c_int32()
    _check(lib.dak_decode_ops(C.byref(m), int(batch), int(context), int(unit_rows), int(chunk_tokens),
                              float(peak_linear), float(peak_attn), None, None, 0, C.byref(n)))
    ops, desc = (dak_op * n.value)(), (dak_op_desc * n.value)()
    _check(lib.dak_decode_ops(C.byref(m), int(batch), int(context), int(unit_rows), int(chunk_tokens),
                              float(peak_linear), float(peak_attn), ops, desc, n.value, C.byref(n)))
    return [dict(kind=o.kind, n_units=o.n_units, unit_bytes=o.unit_bytes, total_bytes=o.total_bytes, T=o.t_comp_s,
                 layer=d.layer, role=ROLES[d.role], M=d.M, K=d.K, flops=d.flops) for o, d in zip(ops, desc)]


def kv_place(seq_lens, page_size: int, max_pages: int, chunk_pages: int, host_units: int):
    """dak_kv_place -> (block table as a numpy int32 [B, max_pages], host pages, HBM pages, host tokens)."""
    import numpy as np
    B = len(seq_lens)
    sl = (C.c_int32 * B)(*[int(x) for x in seq_lens])
    bt = np.zeros((B, max_pages), dtype=np.int32)
    nh, ng, ht = C.c_int32(), C.c_int32(), C.c_int64()
    _check(lib.dak_kv_place(B, sl, int(page_size), int(max_pages), int(chunk_pages), int(host_units),
                            bt.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nh), C.byref(ng), C.byref(ht)))
    return bt, nh.value, ng.value, ht.value


def kv_replace(old_table, seq_lens, page_size: int, max_pages: int, chunk_pages: int, host_units: int,
               host_pool_pages: int, hbm_pool_pages: int):
    """dak_kv_replace -> (new block table numpy int32 [B, max_pages], moves numpy int32 [n, 2])."""
    import numpy as np
    B = len(seq_lens)
    sl = (C.c_int32 * B)(*[int(x) for x in seq_lens])
    old = np.ascontiguousarray(np.asarray(old_table).astype(np.uint32).view(np.int32).reshape(B, max_pages))
    new = np.zeros((B, max_pages), dtype=np.int32)
    mv = np.zeros((B * max_pages, 2), dtype=np.int32)
    n = C.c_int32()
    P = C.POINTER(C.c_int32)
    _check(lib.dak_kv_replace(B, sl, int(page_size), int(max_pages), int(chunk_pages), int(host_units),
                              int(host_pool_pages), int(hbm_pool_pages), old.ctypes.data_as(P), new.ctypes.data_as(P),
                              mv.ctypes.data_as(P), B * max_pages, C.byref(n)))
    return new, mv[:n.value].copy()


def kv_migrate(moves, n_moves, Hkv, page_size, d, k_hbm, v_hbm, k_host, v_host, stream=None):
    _check(lib.dak_kv_migrate(_ptr(moves), int(n_moves), int(Hkv), int(page_size), int(d), _ptr(k_hbm), _ptr(v_hbm),
                              _ptr(k_host), _ptr(v_host), _stream(stream)))


# ------------------------------------------------------------------------------------- calibration
class dak_calib_opts(C.Structure):
    _fields_ = [("n_host", C.c_int32 * 8), ("n_n_host", C.c_int32), ("window", C.c_int32 * 8), ("n_window", C.c_int32),
                ("chunk_bytes", C.c_int32), ("duration_us", C.c_int32), ("reps", C.c_int32), ("op_mb", C.c_int32),
                ("tolerance", C.c_double)]


class dak_calib_result(C.Structure):
    _fields_ = [("n_cta_host", C.c_int32), ("window", C.c_int32), ("host_inflight_bytes", C.c_int64),
                ("hbm_bps", C.c_double), ("link_bps", C.c_double), ("hbm_alone_bps", C.c_double),
                ("host_latency_s", C.c_double)]


_sig("dak_calib_select", C.c_int32, [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32), C.c_double, C.POINTER(C.c_int32), C.POINTER(C.c_int32)])
_sig("dak_calibrate", C.c_int32, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.POINTER(dak_calib_opts),
                                  C.POINTER(dak_calib_result), C.POINTER(C.c_double)])
EXPORTED += ["dak_calib_select", "dak_calibrate"]


def calib_select(table, n_host, window, tolerance: float):
    """dak_calib_select: table [len(n_host)][len(window)][2] (HBM, host B/s) -> (i, j) of the choice."""
    import numpy as np
    t = np.ascontiguousarray(np.asarray(table, dtype=np.float64))
    ni, nw = len(n_host), len(window)
    hs = (C.c_int32 * ni)(*[int(v) for v in n_host])
    ws = (C.c_int32 * nw)(*[int(v) for v in window])
    bi, bj = C.c_int32(), C.c_int32()
    _check(lib.dak_calib_select(t.ctypes.data_as(C.POINTER(C.c_double)), ni, nw, hs, ws, float(tolerance),
                                C.byref(bi), C.byref(bj)))
    return bi.value, bj.value


def calibrate(hbm_buf, hbm_bytes: int, host_dev_ptr, host_bytes: int, n_host=(1, 2, 4, 8, 16),
              window=(1, 2, 4, 6, 8), chunk_bytes: int = 16384, duration_us: int = 300, reps: int = 3,
              tolerance: float = 0.005, op_mb: int = 384):
    """dak_calibrate -> (result dict, table numpy [len(n_host), len(window), 2])."""
    import numpy as np
    o = dak_calib_opts()
    o.n_n_host, o.n_window = len(n_host), len(window)
    for i, v in enumerate(n_host):
        o.n_host[i] = int(v)
    for j, v in enumerate(window):
        o.window[j] = int(v)
    o.chunk_bytes, o.duration_us, o.reps, o.tolerance = int(chunk_bytes), int(duration_us), int(reps), float(tolerance)
    o.op_mb = int(op_mb)
    r = dak_calib_result()
    tab = np.zeros((len(n_host), len(window), 2), dtype=np.float64)
    _check(lib.dak_calibrate(_ptr(hbm_buf), int(hbm_bytes), _ptr(host_dev_ptr), int(host_bytes), C.byref(o), C.byref(r),
                             tab.ctypes.data_as(C.POINTER(C.c_double))))
    return {f: getattr(r, f) for f, _ in dak_calib_result._fields_}, tab


# ------------------------------------------------------------------------------------- host tier
def host_alloc(nbytes: int, write_combined: bool = False, numa_node: int = -1):
    """Pinned + mapped host allocation -> (host_ptr, dev_ptr) ints."""
    hp, dp = C.c_void_p(), C.c_void_p()
    _check(lib.dak_host_alloc(int(nbytes), int(bool(write_combined)), int(numa_node), C.byref(hp), C.byref(dp)))
    return hp.value, dp.value


def host_free(host_ptr: int):
    _check(lib.dak_host_free(host_ptr))


_sig("dak_device_numa_node", C.c_int32, [C.POINTER(C.c_int32)])
EXPORTED += ["dak_device_numa_node"]


def device_numa_node() -> int:
    """NUMA node of the current GPU's PCIe attachment (-1: unknown)."""
    v = C.c_int32()
    _check(lib.dak_device_numa_node(C.byref(v)))
    return v.value


# ------------------------------------------------------------------------------------- linear
def default_kc(M: int, K: int, n_ctas: int = 0) -> int:
    return int(lib.dak_linear_default_kc(int(M), int(K), int(n_ctas)))


def pack_linear(src, rows: int, K: int, kc: int, dst, stream=None):
    _check(lib.dak_pack_linear(_ptr(src), int(rows), int(K), int(kc), _ptr(dst), _stream(stream)))


def launch_cfg(**kw) -> dak_launch_cfg:
    c = dak_launch_cfg()
    for k, v in kw.items():
        setattr(c, k, int(v))
    return c


def linear_args(w_host, w_hbm, M, K, h, kc, N, x, y, bias=None, residual=None, act=ACT_NONE, cfg=None, ldy=0,
                l2_prefetch=None, l2_prefetch_bytes=0, ln_w=None, ln_b=None, ln_stats=None, ln_parts=0, ln_rms=0,
                ln_eps=1e-5, stats_out=None, x_swiglu=0):
    a = dak_linear_args()
    a.w_host = _ptr(w_host)
    a.w_hbm = _ptr(w_hbm)
    a.M, a.K, a.h, a.kc, a.N = int(M), int(K), int(h), int(kc), int(N)
    a.x, a.y = _ptr(x), _ptr(y)
    a.bias, a.residual = _ptr(bias), _ptr(residual)
    a.act = int(act)
    a.cfg = cfg if isinstance(cfg, dak_launch_cfg) else launch_cfg(**(cfg or {}))
    a.ldy = int(ldy)
    a.l2_prefetch, a.l2_prefetch_bytes = _ptr(l2_prefetch), int(l2_prefetch_bytes)
    a.ln_w, a.ln_b, a.ln_stats = _ptr(ln_w), _ptr(ln_b), _ptr(ln_stats)
    a.ln_parts, a.ln_rms, a.ln_eps = int(ln_parts), int(ln_rms), float(ln_eps)
    a.stats_out = _ptr(stats_out)
    a.x_swiglu = int(x_swiglu)
    return a


def linear(args: dak_linear_args, stream=None):
    _check(lib.dak_linear(C.byref(args), _stream(stream)))


_sig("dak_linear_chain", C.c_int32, [C.POINTER(dak_linear_args), C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p])
EXPORTED += ["dak_linear_chain"]


def linear_chain(ops: list, workspace, workspace_bytes: int, stream=None):
    """dak_linear_chain: the ops (dak_linear_args) in one persistent launch; workspace zero-filled."""
    arr = (dak_linear_args * len(ops))(*ops)
    _check(lib.dak_linear_chain(arr, len(ops), _ptr(workspace), int(workspace_bytes), _stream(stream)))


def linear_workspace_size(args: dak_linear_args) -> int:
    return int(lib.dak_linear_workspace_size(C.byref(args)))


def linear_query(args: dak_linear_args) -> dict:
    info = dak_linear_launch_info()
    _check(lib.dak_linear_query(C.byref(args), C.byref(info)))
    return {f: getattr(info, f) for f, _ in dak_linear_launch_info._fields_}


def linear_cta_rows(args: dak_linear_args, cta: int):
    tier, b, e = C.c_int32(), C.c_int64(), C.c_int64()
    _check(lib.dak_linear_cta_rows(C.byref(args), int(cta), C.byref(tier), C.byref(b), C.byref(e)))
    return ("host" if tier.value else "hbm", b.value, e.value)


# ------------------------------------------------------------------------------------- attention
def pack_kv_pages(src, n_blocks: int, page_size: int, d: int, dst, stream=None):
    _check(lib.dak_pack_kv_pages(_ptr(src), int(n_blocks), int(page_size), int(d), _ptr(dst), _stream(stream)))


def attention_args(q, out, k_hbm, v_hbm, k_host, v_host, block_table, seq_lens, B, Hq, Hkv, d, page_size, max_pages,
                   chunk_pages, scale=0.0, workspace=None, workspace_bytes=0, cfg=None, q_row_stride=0, k_new=None,
                   v_new=None, kv_new_stride=0):
    a = dak_attention_args()
    a.q, a.out = _ptr(q), _ptr(out)
    a.k_hbm, a.v_hbm, a.k_host, a.v_host = _ptr(k_hbm), _ptr(v_hbm), _ptr(k_host), _ptr(v_host)
    a.block_table, a.seq_lens = _ptr(block_table), _ptr(seq_lens)
    a.B, a.Hq, a.Hkv, a.d = int(B), int(Hq), int(Hkv), int(d)
    a.page_size, a.max_pages, a.chunk_pages = int(page_size), int(max_pages), int(chunk_pages)
    a.scale = float(scale)
    a.workspace, a.workspace_bytes = _ptr(workspace), int(workspace_bytes)
    a.cfg = cfg if isinstance(cfg, dak_launch_cfg) else launch_cfg(**(cfg or {}))
    a.q_row_stride = int(q_row_stride)
    a.k_new, a.v_new, a.kv_new_stride = _ptr(k_new), _ptr(v_new), int(kv_new_stride)
    return a


def attention_workspace_size(args: dak_attention_args) -> int:
    v = C.c_size_t()
    _check(lib.dak_attention_workspace_size(C.byref(args), C.byref(v)))
    return v.value


def attention(args: dak_attention_args, stream=None):
    _check(lib.dak_attention(C.byref(args), _stream(stream)))


class dak_prefill_args(C.Structure):
    _fields_ = [("q", C.c_void_p), ("out", C.c_void_p), ("k_hbm", C.c_void_p), ("v_hbm", C.c_void_p),
                ("k_host", C.c_void_p), ("v_host", C.c_void_p), ("block_table", C.c_void_p), ("seq_lens", C.c_void_p),
                ("B", C.c_int32), ("T", C.c_int32), ("Hq", C.c_int32), ("Hkv", C.c_int32), ("d", C.c_int32),
                ("page_size", C.c_int32), ("max_pages", C.c_int32), ("scale", C.c_float), ("cfg", dak_launch_cfg),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t)]


_sig("dak_prefill_attention", C.c_int32, [C.POINTER(dak_prefill_args), C.c_void_p])
_sig("dak_prefill_workspace_size", C.c_int32, [C.POINTER(dak_prefill_args), C.POINTER(C.c_size_t)])
EXPORTED += ["dak_prefill_attention", "dak_prefill_workspace_size"]


def prefill_workspace_size(B, Hkv, page_size, max_pages) -> int:
    a = dak_prefill_args()
    a.B, a.Hkv, a.page_size, a.max_pages = int(B), int(Hkv), int(page_size), int(max_pages)
    v = C.c_size_t()
    _check(lib.dak_prefill_workspace_size(C.byref(a), C.byref(v)))
    return v.value


def prefill_attention(q, out, k_hbm, v_hbm, k_host, v_host, block_table, seq_lens, B, T, Hq, Hkv, d, page_size,
                      max_pages, scale=0.0, cfg=None, stream=None, workspace=None, workspace_bytes=0):
    a = dak_prefill_args()
    a.q, a.out = _ptr(q), _ptr(out)
    a.k_hbm, a.v_hbm, a.k_host, a.v_host = _ptr(k_hbm), _ptr(v_hbm), _ptr(k_host), _ptr(v_host)
    a.block_table, a.seq_lens = _ptr(block_table), _ptr(seq_lens)
    a.B, a.T, a.Hq, a.Hkv, a.d = int(B), int(T), int(Hq), int(Hkv), int(d)
    a.page_size, a.max_pages, a.scale = int(page_size), int(max_pages), float(scale)
    a.cfg = cfg if isinstance(cfg, dak_launch_cfg) else launch_cfg(**(cfg or {}))
    a.workspace, a.workspace_bytes = _ptr(workspace), int(workspace_bytes)
    _check(lib.dak_prefill_attention(C.byref(a), _stream(stream)))


def kv_append(k_new, v_new, block_table, positions, B, Hkv, d, page_size, max_pages, k_hbm, v_hbm, k_host, v_host,
              pdl=0, stream=None, row_stride=0):
    _check(lib.dak_kv_append(_ptr(k_new), _ptr(v_new), int(row_stride), _ptr(block_table), _ptr(positions), int(B), int(Hkv), int(d),
                             int(page_size), int(max_pages), _ptr(k_hbm), _ptr(v_hbm), _ptr(k_host), _ptr(v_host),
                             int(pdl), _stream(stream)))


# ------------------------------------------------------------------------------------- layer
MODEL_OPT = 0


class dak_weight(C.Structure):
    _fields_ = [("w_host", C.c_void_p), ("w_hbm", C.c_void_p), ("h", C.c_int64), ("kc", C.c_int32),
                ("n_cta_host", C.c_int32), ("bias", C.c_void_p)]


class dak_layer_args(C.Structure):
    _fields_ = [("model", C.c_int32), ("B", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("ln_eps", C.c_float),
                ("qkv", dak_weight), ("o", dak_weight), ("up", dak_weight), ("down", dak_weight),
                ("ln1_w", C.c_void_p), ("ln1_b", C.c_void_p), ("ln2_w", C.c_void_p), ("ln2_b", C.c_void_p),
                ("x", C.c_void_p), ("scratch", C.c_void_p), ("scratch_bytes", C.c_size_t),
                ("k_hbm", C.c_void_p), ("v_hbm", C.c_void_p), ("k_host", C.c_void_p), ("v_host", C.c_void_p),
                ("block_table", C.c_void_p), ("positions", C.c_void_p), ("seq_lens", C.c_void_p),
                ("page_size", C.c_int32), ("max_pages", C.c_int32), ("chunk_pages", C.c_int32),
                ("tp_rank", C.c_int32), ("tp_size", C.c_int32), ("x_prenormed", C.c_int32),
                ("cfg", dak_launch_cfg), ("attn_cfg", dak_launch_cfg), ("split_qkv", C.c_int32),
                ("reserved2", C.c_int32), ("q", dak_weight), ("k", dak_weight), ("v", dak_weight),
                ("l2_prefetch_bytes", C.c_int64), ("next_w_hbm", C.c_void_p), ("next_w_hbm_bytes", C.c_int64),
                ("fuse_norm", C.c_int32), ("stats_in_parts", C.c_int32), ("stats_in", C.c_void_p),
                ("stats_out", C.c_void_p), ("rope_theta", C.c_float), ("reserved4", C.c_int32), ("comm", C.c_void_p),
                ("next_ln_w", C.c_void_p), ("nvls", C.c_void_p)]


_sig("dak_layernorm", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float,
                                  C.c_int32, C.c_void_p])
_sig("dak_embed", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                              C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p])
_sig("dak_rmsnorm", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_int32,
                                C.c_void_p])
_sig("dak_silu_mul", C.c_int32, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p])
_sig("dak_row_stats", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p])
_sig("dak_layer_scratch_size", C.c_int32, [C.POINTER(dak_layer_args), C.POINTER(C.c_size_t)])
_sig("dak_layer", C.c_int32, [C.POINTER(dak_layer_args), C.c_void_p])
_sig("dak_layer_stats_parts", C.c_int32, [C.POINTER(dak_layer_args), C.POINTER(C.c_int32)])
_sig("dak_rope_kv_append", C.c_int32, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_float, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int32, C.c_void_p])
_sig("dak_comm_unique_id", C.c_int32, [C.c_void_p])
_sig("dak_comm_init", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)])
_sig("dak_comm_destroy", C.c_int32, [C.c_void_p])
_sig("dak_allreduce_residual", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                           C.c_int32, C.c_void_p])
_sig("dak_allreduce_residual_rmsnorm", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                                   C.c_float, C.c_void_p, C.c_int32, C.c_void_p])
EXPORTED += ["dak_layernorm", "dak_rmsnorm", "dak_silu_mul", "dak_embed", "dak_row_stats", "dak_layer_scratch_size", "dak_layer",
             "dak_layer_stats_parts", "dak_rope_kv_append", "dak_comm_unique_id", "dak_comm_init", "dak_comm_destroy",
             "dak_allreduce_residual", "dak_allreduce_residual_rmsnorm"]
MODEL_LLAMA = 1


def rope_kv_append(qkv, row_stride, B, Hq, Hkv, d, positions, rope_theta, block_table, page_size, max_pages, k_hbm,
                   v_hbm, k_host, v_host, pdl=0, stream=None):
    _check(lib.dak_rope_kv_append(_ptr(qkv), int(row_stride), int(B), int(Hq), int(Hkv), int(d), _ptr(positions),
                                  float(rope_theta), _ptr(block_table), int(page_size), int(max_pages), _ptr(k_hbm),
                                  _ptr(v_hbm), _ptr(k_host), _ptr(v_host), int(pdl), _stream(stream)))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.dak_comm_unique_id(buf))
    return buf.raw


def comm_init(uid: bytes, rank: int, world: int) -> int:
    c = C.c_void_p()
    _check(lib.dak_comm_init(C.create_string_buffer(uid, 128), int(rank), int(world), C.byref(c)))
    return c.value


_sig("dak_comm_size", C.c_int32, [C.c_void_p, C.POINTER(C.c_int32)])
_sig("dak_allgather_cols", C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p])
EXPORTED += ["dak_comm_size", "dak_allgather_cols"]


def comm_size(comm) -> int:
    v = C.c_int32()
    _check(lib.dak_comm_size(comm, C.byref(v)))
    return v.value


def allgather_cols(comm, send, recv, scratch, N, Ml, stream=None):
    _check(lib.dak_allgather_cols(comm, _ptr(send), _ptr(recv), _ptr(scratch), int(N), int(Ml), _stream(stream)))


_sig("dak_nvls_create", C.c_int32, [C.c_void_p, C.c_size_t, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)])
_sig("dak_nvls_destroy", C.c_int32, [C.c_void_p])
_sig("dak_nvls_local", C.c_void_p, [C.c_void_p])
_sig("dak_nvls_residual_rmsnorm", C.c_int32, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                              C.c_float, C.c_void_p, C.c_void_p])
EXPORTED += ["dak_nvls_create", "dak_nvls_destroy", "dak_nvls_local", "dak_nvls_residual_rmsnorm"]


def nvls_create(comm, nbytes: int, max_rows: int):
    """-> (handle, local window pointer); raises DakError EUNSUPPORTED without a multicast team."""
    h, buf = C.c_void_p(), C.c_void_p()
    _check(lib.dak_nvls_create(comm, int(nbytes), int(max_rows), C.byref(h), C.byref(buf)))
    return h.value, buf.value


def nvls_destroy(h):
    _check(lib.dak_nvls_destroy(h))


def nvls_residual_rmsnorm(h, offset, x, rows, cols, norm_w, eps, y_norm, stream=None):
    _check(lib.dak_nvls_residual_rmsnorm(h, int(offset), _ptr(x), int(rows), int(cols), _ptr(norm_w), float(eps),
                                         _ptr(y_norm), _stream(stream)))


def comm_destroy(comm):
    _check(lib.dak_comm_destroy(comm))


def allreduce_residual(comm, partial, x, rows, cols, stats_out=None, pdl=0, stream=None):
    _check(lib.dak_allreduce_residual(comm, _ptr(partial), _ptr(x), int(rows), int(cols), _ptr(stats_out), int(pdl),
                                      _stream(stream)))


def allreduce_residual_rmsnorm(comm, partial, x, rows, cols, norm_w, eps, y_norm, pdl=0, stream=None):
    _check(lib.dak_allreduce_residual_rmsnorm(comm, _ptr(partial), _ptr(x), int(rows), int(cols), _ptr(norm_w),
                                              float(eps), _ptr(y_norm), int(pdl), _stream(stream)))


def weight(w_host, w_hbm, h, kc, bias=None, n_cta_host=0) -> dak_weight:
    return dak_weight(_ptr(w_host), _ptr(w_hbm), int(h), int(kc), int(n_cta_host), _ptr(bias))


def layernorm(x, w, b, y, rows, cols, eps=1e-5, pdl=0, stream=None):
    _check(lib.dak_layernorm(_ptr(x), _ptr(w), _ptr(b), _ptr(y), int(rows), int(cols), float(eps), int(pdl),
                             _stream(stream)))


def embed(tokens, positions, tok_emb, pos_emb, B, hidden, pos_offset, x, pdl=0, stream=None, stats_out=None):
    _check(lib.dak_embed(_ptr(tokens), _ptr(positions), _ptr(tok_emb), _ptr(pos_emb), int(B), int(hidden),
                         int(pos_offset), _ptr(x), _ptr(stats_out), int(pdl), _stream(stream)))


def rmsnorm(x, w, y, rows, cols, eps=1e-5, pdl=0, stream=None):
    _check(lib.dak_rmsnorm(_ptr(x), _ptr(w), _ptr(y), int(rows), int(cols), float(eps), int(pdl), _stream(stream)))


def silu_mul(gu, out, rows, F, pdl=0, stream=None):
    _check(lib.dak_silu_mul(_ptr(gu), _ptr(out), int(rows), int(F), int(pdl), _stream(stream)))


def row_stats(x, rows, cols, stats_out, ld=0, pdl=0, stream=None):
    _check(lib.dak_row_stats(_ptr(x), int(rows), int(cols), int(ld), _ptr(stats_out), int(pdl), _stream(stream)))


def layer_stats_parts(args: dak_layer_args) -> int:
    v = C.c_int32()
    _check(lib.dak_layer_stats_parts(C.byref(args), C.byref(v)))
    return v.value


def layer_scratch_size(args: dak_layer_args) -> int:
    v = C.c_size_t()
    _check(lib.dak_layer_scratch_size(C.byref(args), C.byref(v)))
    return v.value


def layer(args: dak_layer_args, stream=None):
    _check(lib.dak_layer(C.byref(args), _stream(stream)))


_sig("dak_linear_choose_kc", C.c_int32, [C.c_int64, C.c_int64])
EXPORTED += ["dak_linear_choose_kc"]


def choose_kc(rows_per_cta: int, K: int) -> int:
    return int(lib.dak_linear_choose_kc(int(rows_per_cta), int(K)))
