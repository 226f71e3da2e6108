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
                ("host_capacity_bytes", C.c_int64)]


class dak_op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("n_units", C.c_int64), ("unit_bytes", C.c_int64),
                ("total_bytes", C.c_int64), ("t_comp_s", C.c_double)]


class dak_op_plan(C.Structure):
    _fields_ = [("host_units", C.c_int64), ("host_bytes", C.c_int64), ("ratio", C.c_double), ("phase", C.c_int32),
                ("reserved", C.c_int32), ("latency_s", C.c_double)]


class dak_launch_cfg(C.Structure):
    _fields_ = [("n_cta_host", C.c_int32), ("n_cta_hbm", C.c_int32), ("window", C.c_int32), ("stages", C.c_int32),
                ("congestion_control", C.c_int32), ("pdl", C.c_int32), ("force_path", C.c_int32),
                ("reserved", C.c_int32)]


class dak_linear_args(C.Structure):
    _fields_ = [("w_host", C.c_void_p), ("w_hbm", C.c_void_p), ("M", C.c_int64), ("K", C.c_int64), ("h", C.c_int64),
                ("kc", C.c_int32), ("N", C.c_int32), ("x", C.c_void_p), ("y", C.c_void_p), ("bias", C.c_void_p),
                ("residual", C.c_void_p), ("act", C.c_int32), ("reserved", C.c_int32), ("cfg", dak_launch_cfg)]


class dak_linear_launch_info(C.Structure):
    _fields_ = [("grid", C.c_int32), ("n_cta_host", C.c_int32), ("n_cta_hbm", C.c_int32), ("threads", C.c_int32),
                ("stages_hbm", C.c_int32), ("window_host", C.c_int32), ("smem_bytes", C.c_int32), ("path", C.c_int32),
                ("rows_per_cta_host_max", C.c_int64), ("rows_per_cta_hbm_max", C.c_int64),
                ("hbm_bytes", C.c_int64), ("host_bytes", C.c_int64)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("dak_last_error", C.c_char_p, [])
_sig("dak_version", C.c_char_p, [])
_sig("dak_device_sms", C.c_int32, [C.POINTER(C.c_int32)])
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

EXPORTED = ["dak_last_error", "dak_version", "dak_device_sms", "dak_plan_ratios", "dak_host_alloc", "dak_host_free",
            "dak_linear_packed_bytes", "dak_pack_linear", "dak_linear_default_kc", "dak_linear_query",
            "dak_linear_cta_rows", "dak_linear"]


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


def device_sms() -> int:
    v = C.c_int32()
    _check(lib.dak_device_sms(C.byref(v)))
    return v.value


# ------------------------------------------------------------------------------------- planner
def plan_ratios(hw: dict, ops: list, y_req_bytes: int, mode: int = PLAN_EXACT):
    """dak_plan_ratios: hw = {hbm_bps, link_bps, host_dram_bps, host_capacity_bytes};
    ops = [{kind, n_units, unit_bytes, total_bytes, T}]. Returns (list of plan dicts, objective)."""
    h = dak_hw(float(hw["hbm_bps"]), float(hw["link_bps"]), float(hw.get("host_dram_bps", hw["link_bps"])),
               int(hw.get("host_capacity_bytes", -1)))
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


# ------------------------------------------------------------------------------------- host tier
def host_alloc(nbytes: int, write_combined: bool = False, numa_node: int = -1):
    """Pinned + mapped host allocation -> (host_ptr, dev_ptr) ints."""
    hp, dp = C.c_void_p(), C.c_void_p()
    _check(lib.dak_host_alloc(int(nbytes), int(bool(write_combined)), int(numa_node), C.byref(hp), C.byref(dp)))
    return hp.value, dp.value


def host_free(host_ptr: int):
    _check(lib.dak_host_free(host_ptr))


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


def linear_args(w_host, w_hbm, M, K, h, kc, N, x, y, bias=None, residual=None, act=ACT_NONE, cfg=None):
    a = dak_linear_args()
    a.w_host = _ptr(w_host)
    a.w_hbm = _ptr(w_hbm)
    a.M, a.K, a.h, a.kc, a.N = int(M), int(K), int(h), int(kc), int(N)
    a.x, a.y = _ptr(x), _ptr(y)
    a.bias, a.residual = _ptr(bias), _ptr(residual)
    a.act = int(act)
    a.cfg = cfg if isinstance(cfg, dak_launch_cfg) else launch_cfg(**(cfg or {}))
    return a


def linear(args: dak_linear_args, stream=None):
    _check(lib.dak_linear(C.byref(args), _stream(stream)))


def linear_query(args: dak_linear_args) -> dict:
    info = dak_linear_launch_info()
    _check(lib.dak_linear_query(C.byref(args), C.byref(info)))
    return {f: getattr(info, f) for f, _ in dak_linear_launch_info._fields_}


def linear_cta_rows(args: dak_linear_args, cta: int):
    tier, b, e = C.c_int32(), C.c_int64(), C.c_int64()
    _check(lib.dak_linear_cta_rows(C.byref(args), int(cta), C.byref(tier), C.byref(b), C.byref(e)))
    return ("host" if tier.value else "hbm", b.value, e.value)
