"""ctypes binding of libtdpipe.so (include/tdpipe.h) -- argument marshalling only.

Every step of the hot path runs inside the C/CUDA library; this module only
converts numpy arrays / Python ints to the C ABI and back.  If the shared
library is missing, importing this module raises (there is no fallback path).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDPIPE_LIB", os.path.join(_HERE, "libtdpipe.so"))

TD_OK, TD_EINVAL, TD_ENOMEM, TD_ECUDA, TD_ENCCL, TD_ERANGE, TD_ESTATE = 0, -1, -2, -3, -4, -5, -6
TD_POLICY_TDPIPE, TD_POLICY_PPSB_PRIO, TD_POLICY_PPSB_ALT, TD_POLICY_PPHB = 0, 1, 2, 3
TD_EXEC_CUDA, TD_EXEC_NULL = 0, 1
TD_BATCH_PREFILL, TD_BATCH_DECODE = 0, 1
TD_HANDOFF_PEER, TD_HANDOFF_NCCL = 0, 1

# int32 (*)(void* user, const void* send, void* recv, size_t bytes) -- include/tdpipe.h td_allgather_fn
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class td_model_shape(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_ffn", C.c_int32), ("vocab", C.c_int32),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("max_seq_len", C.c_int32)]


class td_options(C.Structure):
    _fields_ = [("executor", C.c_int32), ("device", C.c_int32),
                ("block_size", C.c_int32), ("kv_blocks", C.c_int64), ("hbm_reserve_frac", C.c_double),
                ("prefill_token_budget", C.c_int32), ("max_batch_seqs", C.c_int32),
                ("fp_stride", C.c_int32), ("fp_horizon", C.c_int32), ("policy", C.c_int32),
                ("steal", C.c_int32), ("alg1_check_before_launch", C.c_int32),
                ("eq2_bubble_scale", C.c_int32), ("weight_seed", C.c_uint64),
                ("profile_csv", C.c_char_p), ("log_decisions", C.c_int32), ("record_logits", C.c_int32),
                ("world_size", C.c_int32), ("rank", C.c_int32), ("nccl_ids", C.c_void_p),
                ("p2d_kv_permille", C.c_int32), ("d2p_finish_permille", C.c_int32), ("hb_tokens", C.c_int32),
                ("handoff", C.c_int32), ("allgather", ALLGATHER_FN), ("allgather_user", C.c_void_p),
                ("hbm_peak_gbs", C.c_double), ("tc_peak_tflops", C.c_double),
                ("decode_chain", C.c_int32)]


class td_run_stats(C.Structure):
    _fields_ = [("n_requests", C.c_int64), ("prompt_tokens", C.c_int64), ("generated_tokens", C.c_int64),
                ("makespan_ns", C.c_int64), ("gen_tokens_per_s", C.c_double),
                ("total_tokens_per_s", C.c_double), ("bubble_frac", C.c_double),
                ("n_microbatches", C.c_int64), ("n_prefill_mb", C.c_int64), ("n_decode_mb", C.c_int64),
                ("n_p2d", C.c_int64), ("n_d2p", C.c_int64), ("n_stolen", C.c_int64),
                ("n_evicted", C.c_int64), ("gpu_launches", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("busy_ns", C.c_int64 * 8), ("ideal_ns", C.c_double),
                ("alg_bytes", C.c_double), ("alg_flops", C.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "busy_ns"}
        d["busy_ns"] = list(self.busy_ns)
        return d


class td_batch(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_seqs", C.c_int32), ("seq_slot", C.POINTER(C.c_int32)),
                ("q_start", C.POINTER(C.c_int32)), ("q_len", C.POINTER(C.c_int32)),
                ("block_table", C.POINTER(C.c_int32)), ("max_blocks", C.c_int32)]


EXPORTS = ["td_default_options", "td_create", "td_destroy", "td_last_error", "td_submit", "td_upload",
           "td_run", "td_get_output", "td_get_outputs", "td_get_logits", "td_reset", "td_stage_forward",
           "td_kv_reset", "td_profile", "td_load_profile", "td_get_log", "td_info", "td_set_timing",
           "td_get_timing", "td_nccl_ids", "td_test_gemm", "td_test_chain_mlp", "td_bench_gemm", "td_bench_attn", "td_simulate", "td_write_trace",
           "td_get_weight", "td_bench_step", "td_get_launch_bytes"]


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(f"libtdpipe.so not built ({path}); run `python -m paper_2506_10470_b200.build`")
    lib = C.CDLL(path)
    P = C.POINTER
    lib.td_default_options.argtypes = [P(td_options)]
    lib.td_default_options.restype = None
    lib.td_create.argtypes = [P(td_model_shape), C.c_int32, P(td_options), P(C.c_void_p)]
    lib.td_destroy.argtypes = [C.c_void_p]
    lib.td_destroy.restype = None
    lib.td_last_error.argtypes = [C.c_void_p]
    lib.td_last_error.restype = C.c_char_p
    lib.td_submit.argtypes = [C.c_void_p, P(C.c_int32), C.c_int32, C.c_int32, C.c_int32]
    lib.td_submit.restype = C.c_int64
    lib.td_upload.argtypes = [C.c_void_p]
    lib.td_run.argtypes = [C.c_void_p, P(td_run_stats)]
    lib.td_get_output.argtypes = [C.c_void_p, C.c_int64, P(C.c_int32), C.c_int32, P(C.c_int32)]
    lib.td_get_outputs.argtypes = [C.c_void_p, P(C.c_int32), C.c_int32, C.c_int32, P(C.c_int32)]
    lib.td_get_launch_bytes.argtypes = [C.c_void_p, C.c_char_p, P(C.c_double), C.c_int64, P(C.c_int64)]
    lib.td_bench_step.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_double),
                                  P(C.c_double)]
    lib.td_get_weight.argtypes = [C.c_void_p, C.c_int32, P(C.c_uint16), C.c_int64, P(C.c_int64), P(C.c_int64)]
    lib.td_get_logits.argtypes = [C.c_void_p, C.c_int64, P(C.c_float), C.c_int64, P(C.c_int32)]
    lib.td_reset.argtypes = [C.c_void_p]
    lib.td_stage_forward.argtypes = [C.c_void_p, C.c_int32, P(td_batch), C.c_void_p, C.c_void_p]
    lib.td_kv_reset.argtypes = [C.c_void_p]
    lib.td_profile.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32, C.c_int32]
    lib.td_load_profile.argtypes = [C.c_void_p, C.c_char_p]
    lib.td_get_log.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, P(C.c_size_t)]
    lib.td_info.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int32), P(C.c_int64), P(C.c_int64)]
    lib.td_set_timing.argtypes = [C.c_void_p, C.c_int32]
    lib.td_get_timing.argtypes = [C.c_void_p, C.c_char_p, P(C.c_int64), P(C.c_double), P(C.c_double),
                                  P(C.c_double)]
    lib.td_nccl_ids.argtypes = [C.c_void_p]
    lib.td_bench_gemm.argtypes = [C.c_int32] * 8 + [P(C.c_float)]
    lib.td_bench_attn.argtypes = [C.c_int32, C.c_int32, P(C.c_int32)] + [C.c_int32] * 6 + [P(C.c_float)]
    lib.td_simulate.argtypes = [C.c_void_p, P(td_run_stats), C.c_int64]
    lib.td_write_trace.argtypes = [C.c_void_p, C.c_char_p]
    lib.td_test_gemm.argtypes = [C.c_int32, P(C.c_uint16), P(C.c_uint16), C.c_int32, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_int32, P(C.c_float)]
    lib.td_test_chain_mlp.argtypes = [C.c_int32, P(C.c_float), P(C.c_uint16), P(C.c_uint16), P(C.c_uint16),
                                      C.c_int32, C.c_int32, C.c_int32, C.c_float, P(C.c_uint16), P(C.c_uint16),
                                      P(C.c_float)]
    for f in EXPORTS:
        if f not in ("td_default_options", "td_destroy", "td_last_error", "td_submit"):
            getattr(lib, f).restype = C.c_int32
    return lib


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


class TDError(RuntimeError):
    pass


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def make_shape(shape) -> td_model_shape:
    return td_model_shape(shape.n_layers, shape.d_model, shape.n_heads, shape.n_kv_heads, shape.d_ffn,
                          shape.vocab, float(shape.rope_theta), float(shape.rms_eps), shape.max_seq_len)


def make_allgather(gather):
    """Wrap `gather(bytes) -> list[bytes]` (this rank's bytes in, every rank's
    bytes out in rank order -- e.g. torch.distributed.all_gather_object) as the
    td_allgather_fn callback of td_options.allgather."""
    def cb(user, send, recv, nbytes):
        try:
            parts = gather(C.string_at(send, nbytes))
            buf = b"".join(parts)
            C.memmove(recv, buf, len(buf))
            return 0
        except Exception:   # no exception may cross the C ABI
            import traceback
            traceback.print_exc()
            return -1
    return ALLGATHER_FN(cb)


def default_options(**kw) -> td_options:
    o = td_options()
    lib().td_default_options(C.byref(o))
    for k, v in kw.items():
        if k == "profile_csv" and isinstance(v, str):
            v = v.encode()
        if k == "allgather" and not isinstance(v, ALLGATHER_FN):
            v = make_allgather(v)
        setattr(o, k, v)
    return o


class TDPipe:
    """Owner of one td_ctx.  Methods map 1:1 onto the C ABI."""

    def __init__(self, shape, n_stages: int = 1, **opts):
        self.shape = shape
        self._keep = []
        o = default_options(**opts)
        self._keep.append(o.profile_csv)
        self._keep.append(o)   # holds the allgather callback, which must outlive the ctx (td_destroy calls it)
        self.ctx = C.c_void_p()
        st = lib().td_create(C.byref(make_shape(shape)), int(n_stages), C.byref(o), C.byref(self.ctx))
        if st != TD_OK:
            raise TDError(f"td_create failed ({st}): {lib().td_last_error(None).decode()}")
        self.n_stages = n_stages

    def close(self):
        if self.ctx:
            lib().td_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != TD_OK:
            raise TDError(f"{what} failed ({st}): {lib().td_last_error(self.ctx).decode()}")

    def td_submit(self, prompt: Sequence[int], predicted_len: int, max_new_tokens: int) -> int:
        p = _i32(prompt)
        rid = lib().td_submit(self.ctx, _ptr(p, C.c_int32), len(p), int(predicted_len), int(max_new_tokens))
        if rid < 0:
            self._check(int(rid), "td_submit")
        return int(rid)

    def submit_workload(self, wl) -> None:
        for r in wl.requests:
            self.td_submit(r.prompt, r.predicted_len, r.max_new_tokens)

    def td_upload(self):
        self._check(lib().td_upload(self.ctx), "td_upload")

    def td_run(self) -> dict:
        st = td_run_stats()
        self._check(lib().td_run(self.ctx, C.byref(st)), "td_run")
        return st.as_dict()

    def td_simulate(self, host_return_ns: int = 0) -> dict:
        st = td_run_stats()
        self._check(lib().td_simulate(self.ctx, C.byref(st), int(host_return_ns)), "td_simulate")
        return st.as_dict()

    def td_write_trace(self, path: str):
        self._check(lib().td_write_trace(self.ctx, path.encode()), "td_write_trace")

    def td_get_output(self, rid: int) -> np.ndarray:
        n = C.c_int32(0)
        lib().td_get_output(self.ctx, int(rid), None, 0, C.byref(n))
        buf = np.zeros(max(n.value, 1), dtype=np.int32)
        self._check(lib().td_get_output(self.ctx, int(rid), _ptr(buf, C.c_int32), len(buf), C.byref(n)),
                    "td_get_output")
        return buf[: n.value].copy()

    def td_get_outputs(self, n_requests: int, stride: int):
        out = np.zeros((n_requests, stride), dtype=np.int32)
        n = np.zeros(n_requests, dtype=np.int32)
        self._check(lib().td_get_outputs(self.ctx, _ptr(out, C.c_int32), n_requests, stride, _ptr(n, C.c_int32)),
                    "td_get_outputs")
        return out, n

    def td_bench_step(self, kind: int, n_seqs: int, length: int, iters: int = 10):
        """(mean step us, speed-of-light us) of one synthetic micro-batch; per-kernel
        timing is then readable with td_get_timing."""
        us, ideal = C.c_double(), C.c_double()
        self._check(lib().td_bench_step(self.ctx, int(kind), int(n_seqs), int(length), int(iters), C.byref(us),
                                        C.byref(ideal)), "td_bench_step")
        return us.value, ideal.value

    def td_get_launch_bytes(self, name: str) -> np.ndarray:
        """Per-launch algorithmic bytes of kernel class `name` (timed runs), launch order."""
        n = C.c_int64()
        self._check(lib().td_get_launch_bytes(self.ctx, name.encode(), None, 0, C.byref(n)), "td_get_launch_bytes")
        out = np.zeros(max(n.value, 1), dtype=np.float64)
        self._check(lib().td_get_launch_bytes(self.ctx, name.encode(), _ptr(out, C.c_double), out.size, C.byref(n)),
                    "td_get_launch_bytes")
        return out[: n.value]

    def td_get_weight(self, tensor_id: int) -> np.ndarray:
        """bf16 bit patterns (uint16) of F9 tensor `tensor_id`, logical [rows, cols]."""
        r, c = C.c_int64(), C.c_int64()
        lib().td_get_weight(self.ctx, int(tensor_id), None, 0, C.byref(r), C.byref(c))
        buf = np.zeros(max(r.value * c.value, 1), dtype=np.uint16)
        self._check(lib().td_get_weight(self.ctx, int(tensor_id), _ptr(buf, C.c_uint16), buf.size, C.byref(r),
                                        C.byref(c)), "td_get_weight")
        return buf[: r.value * c.value].reshape(r.value, c.value)

    def td_get_logits(self, rid: int) -> np.ndarray:
        ns = C.c_int32(0)
        lib().td_get_logits(self.ctx, int(rid), None, 0, C.byref(ns))
        buf = np.zeros((max(ns.value, 1), self.shape.vocab), dtype=np.float32)
        self._check(lib().td_get_logits(self.ctx, int(rid), _ptr(buf, C.c_float), buf.size, C.byref(ns)),
                    "td_get_logits")
        return buf[: ns.value].copy()

    def td_reset(self):
        self._check(lib().td_reset(self.ctx), "td_reset")

    def td_kv_reset(self):
        self._check(lib().td_kv_reset(self.ctx), "td_kv_reset")

    def td_stage_forward(self, stage: int, kind: int, q_start, q_len, block_table: np.ndarray, inp: np.ndarray):
        qs, ql = _i32(q_start), _i32(q_len)
        bt = _i32(block_table)
        n = len(qs)
        slots = _i32(np.arange(n))
        b = td_batch(kind, n, _ptr(slots, C.c_int32), _ptr(qs, C.c_int32), _ptr(ql, C.c_int32),
                     _ptr(bt, C.c_int32), bt.shape[1])
        T = int(ql.sum())
        if stage == 0:
            inp = _i32(inp)
        else:
            inp = np.ascontiguousarray(inp, dtype=np.float32)
        if stage == self.n_stages - 1:
            out = np.zeros((n, self.shape.vocab), dtype=np.float32)
        else:
            out = np.zeros((T, self.shape.d_model), dtype=np.float32)
        self._check(lib().td_stage_forward(self.ctx, int(stage), C.byref(b), inp.ctypes.data_as(C.c_void_p),
                                           out.ctypes.data_as(C.c_void_p)), "td_stage_forward")
        return out

    def td_profile(self, out_csv: Optional[str], b_max: int, k_max: int, ctx_len: int):
        self._check(lib().td_profile(self.ctx, out_csv.encode() if out_csv else None, b_max, k_max, ctx_len),
                    "td_profile")

    def td_load_profile(self, csv: str):
        self._check(lib().td_load_profile(self.ctx, csv.encode()), "td_load_profile")

    def td_get_log(self) -> str:
        need = C.c_size_t(0)
        lib().td_get_log(self.ctx, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value + 1)
        self._check(lib().td_get_log(self.ctx, buf, need.value, C.byref(need)), "td_get_log")
        return buf.raw[: need.value].decode()

    def td_info(self) -> dict:
        kb, ns, wb, kvb = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64()
        self._check(lib().td_info(self.ctx, C.byref(kb), C.byref(ns), C.byref(wb), C.byref(kvb)), "td_info")
        return dict(kv_blocks=kb.value, n_stages=ns.value, weight_bytes=wb.value, kv_bytes_per_block=kvb.value)

    def td_set_timing(self, on: bool):
        self._check(lib().td_set_timing(self.ctx, int(on)), "td_set_timing")

    def td_get_timing(self, name: str) -> dict:
        n, ms, b, f = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        self._check(lib().td_get_timing(self.ctx, name.encode(), C.byref(n), C.byref(ms), C.byref(b), C.byref(f)),
                    "td_get_timing")
        return dict(launches=n.value, ms=ms.value, bytes=b.value, flops=f.value)


def td_nccl_ids() -> bytes:
    buf = C.create_string_buffer(256)
    st = lib().td_nccl_ids(buf)
    if st != TD_OK:
        raise TDError(f"td_nccl_ids failed: {st}")
    return buf.raw


def td_test_gemm(A_bits: np.ndarray, W_bits: np.ndarray, impl: int = 0, splits: int = 1, device: int = 0):
    """Kernel unit test: fp32 [T, N] = A . W^T for bf16 bit patterns (uint16)."""
    A = np.ascontiguousarray(A_bits, dtype=np.uint16)
    W = np.ascontiguousarray(W_bits, dtype=np.uint16)
    T, K = A.shape
    N = W.shape[0]
    out = np.zeros((T, N), dtype=np.float32)
    st = lib().td_test_gemm(device, _ptr(A, C.c_uint16), _ptr(W, C.c_uint16), T, N, K, impl, splits,
                            _ptr(out, C.c_float))
    if st != TD_OK:
        raise TDError(f"td_test_gemm failed: {st}")
    return out


def td_bench_gemm(T: int, N: int, K: int, splits: int = 1, decode: bool = True, iters: int = 50, copies: int = 4,
                  device: int = 0) -> float:
    """Average device microseconds per tcgen05 GEMM call (weights streamed from HBM)."""
    us = C.c_float(0)
    st = lib().td_bench_gemm(device, T, N, K, splits, int(decode), iters, copies, C.byref(us))
    if st != TD_OK:
        raise TDError(f"td_bench_gemm failed: {st}")
    return us.value


def td_bench_attn(ctx, H: int, Hkv: int, hd: int, iters: int = 50, device: int = 0, split: int = 0,
                  impl: int = 0) -> float:
    """Average device microseconds per decode-attention launch over context
    lengths `ctx` (the engine's launch plan, or `split`-token splits)."""
    c = np.ascontiguousarray(ctx, dtype=np.int32)
    us = C.c_float(0)
    st = lib().td_bench_attn(device, len(c), _ptr(c, C.c_int32), H, Hkv, hd, iters, int(split), int(impl),
                             C.byref(us))
    if st != TD_OK:
        raise TDError(f"td_bench_attn failed: {st}")
    return us.value


def td_test_chain_mlp(x0: np.ndarray, g_bits: np.ndarray, Wgu_bits: np.ndarray, Wd_bits: np.ndarray,
                      eps: float = 1e-5, device: int = 0):
    """Kernel unit test of the decode chain on one MLP block: returns
    (a bf16 bits [T, d], h bf16 bits [T, F], x fp32 [T, d])."""
    x0 = np.ascontiguousarray(x0, dtype=np.float32)
    g = np.ascontiguousarray(g_bits, dtype=np.uint16)
    Wgu = np.ascontiguousarray(Wgu_bits, dtype=np.uint16)
    Wd = np.ascontiguousarray(Wd_bits, dtype=np.uint16)
    T, d = x0.shape
    F = Wd.shape[1]
    a = np.zeros((T, d), np.uint16)
    h = np.zeros((T, F), np.uint16)
    x = np.zeros((T, d), np.float32)
    st = lib().td_test_chain_mlp(device, _ptr(x0, C.c_float), _ptr(g, C.c_uint16), _ptr(Wgu, C.c_uint16),
                                 _ptr(Wd, C.c_uint16), T, d, F, eps, _ptr(a, C.c_uint16), _ptr(h, C.c_uint16),
                                 _ptr(x, C.c_float))
    if st != TD_OK:
        raise TDError(f"td_test_chain_mlp failed: {st}")
    return a, h, x
