"""Thin ctypes binding of libelis (include/elis.h, include/elis_ops.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Device arrays are passed as raw pointers (``tensor.data_ptr()``),
streams as ``torch.cuda.current_stream().cuda_stream``.  There is no CPU
fallback: if the library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import inputs

_HERE = os.path.dirname(os.path.abspath(__file__))
# ELIS_LIB selects an alternative in-tree build (A/B kernel experiments); default libelis.so
LIB_PATH = os.path.join(_HERE, os.environ.get("ELIS_LIB", "libelis.so"))

ELIS_OK = 0
ABI_VERSION = 5  # include/elis.h ELIS_ABI_VERSION
STATUS = {0: "ok", 1: "invalid argument", 2: "config", 3: "unsupported device", 4: "oom", 5: "cuda",
          6: "nccl", 7: "device input", 8: "peer timeout"}
POLICY_ISRTF, POLICY_FCFS = 0, 1
EPI_BIAS_BF16, EPI_BIAS_GELU_BF16, EPI_BIAS_RESID_F32 = 0, 1, 2
PRECISION = {"auto": 0, "fp8": 1, "fp16": 2, "bf16": 3}  # elis_precision (auto: fp16 for head dim 64, else bf16)
RESIDUAL = {None: 0, True: 1, False: 2}  # elis_residual: auto / fp16 stream / fp32 stream

_vp, _i32, _i64, _u32, _f32, _sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                    ctypes.c_float, ctypes.c_size_t)


class ElisConfig(ctypes.Structure):
    _fields_ = [("abi_version", _i32), ("vocab_size", _i32), ("max_position", _i32), ("type_vocab_size", _i32),
                ("num_layers", _i32), ("hidden", _i32), ("num_heads", _i32), ("intermediate", _i32),
                ("ln_eps", _f32), ("pooling", _i32), ("head_layers", _i32), ("head_hidden", _i32),
                ("head_predicts_total", _i32), ("max_tokens", _i32), ("max_requests", _i32), ("device", _i32),
                ("precision", _i32), ("cls_last_layer", _i32), ("residual_stream", _i32)]


class ElisStarvation(ctypes.Structure):
    _fields_ = [("windows_waited", _vp), ("boost_after", _i32), ("boost_amount", _f32), ("preempt_margin", _f32)]


class ElisPreempt(ctypes.Structure):
    _fields_ = [("policy", _i32), ("allow_preempt", _i32), ("order", _vp), ("running", _vp),
                ("out_preempted", _vp), ("out_count", _vp), ("out_nan_count", _vp),
                ("starvation", ctypes.POINTER(ElisStarvation))]


def _preempt(policy, allow_preempt, order, running, out_preempted, out_count, out_nan_count,
             windows_waited=None, boost_after=1, boost_amount=0.0, preempt_margin=0.0):
    """elis_preempt (+ elis_starvation when aging or a margin is requested); the returned
    struct keeps its starvation struct alive."""
    pre = ElisPreempt(policy, int(allow_preempt), _ptr(order), _ptr(running), _ptr(out_preempted),
                      _ptr(out_count), _ptr(out_nan_count), None)
    if windows_waited is not None or boost_amount or preempt_margin:
        sv = ElisStarvation(_ptr(windows_waited), int(boost_after), float(boost_amount), float(preempt_margin))
        pre._sv = sv
        pre.starvation = ctypes.pointer(sv)
    return pre


class ElisError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libelis.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ElisError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "elis_abi_version": (_i32, []),
        "elis_weight_count": (_sz, [_vp]),
        "elis_predictor_create": (_i32, [_vp, _vp, _sz, ctypes.POINTER(_vp)]),
        "elis_predictor_destroy": (None, [_vp]),
        "elis_predict_remaining": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp]),
        "elis_predict_remaining_dev": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        "elis_isrtf_select": (_i32, [_vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]),
        "elis_nccl_unique_id": (_i32, [_vp]),
        "elis_dist_attach": (_i32, [_vp, _i32, _i32, _vp]),
        "elis_isrtf_select_dist": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
        "elis_peer_export": (_i32, [_vp, _i32, _i32, _vp]),
        "elis_peer_attach": (_i32, [_vp, _vp]),
        "elis_peer_attach_local": (_i32, [_vp, _i32]),
        "elis_assign_nodes": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp]),
        "elis_isrtf_select_nodes": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
        "elis_iteration_host": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp,
                                       _vp, _vp, _vp]),
        "elis_predict_remaining_dist": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp]),
        "elis_iteration_table_host": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp,
                                             _vp]),
        "elis_cost_split": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp]),
        "elis_arena_create": (_i32, [_i32, _i32, _vp]),
        "elis_arena_destroy": (None, [_vp]),
        "elis_arena_set_prompts": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp]),
        "elis_arena_append": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp]),
        "elis_arena_gather": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
        "elis_arena_sync_status": (_i32, [_vp, _vp]),
        "elis_sync_status": (_i32, [_vp]),
        "elis_last_device_error_bits": (_u32, [_vp]),
        "elis_status_string": (ctypes.c_char_p, [_i32]),
        "elis_last_error": (ctypes.c_char_p, []),
        "elis_get_hidden": (_i32, [_vp, _vp, _i64, _vp]),
        "elis_launch_count": (ctypes.c_uint64, [_vp]),
        "elis_profile_enable": (_i32, [_vp, _i32]),
        "elis_profile_read": (_i32, [_vp, _vp, _vp, _vp, _i32]),
        "elis_op_gemm": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
        "elis_op_gemm_f16": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
        "elis_op_gemm_ln": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _f32, _vp, _i32, _i32, _i32, _vp]),
        "elis_op_quant_rows_e4m3": (_i32, [_vp, _i32, _i32, _vp, _vp, _f32, _vp]),
        "elis_op_gemm_f8": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _f32, _vp]),
        "elis_op_gemm_ln16": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _vp]),
        "elis_op_gemm_ln_f8": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _vp, _f32, _i32, _i32, _i32, _vp]),
        "elis_op_attention": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp, _vp]),
        "elis_op_attention_f16": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp, _vp]),
        "elis_op_layernorm": (_i32, [_vp, _vp, _vp, _f32, _i64, _i32, _vp, _vp, _vp]),
        "elis_op_fc_f32": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int, what: str = ""):
    if status != ELIS_OK:
        detail = lib().elis_last_error().decode(errors="replace")
        raise ElisError(f"{what}: {STATUS.get(status, status)} ({detail})")


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_config(cfg: inputs.EncoderConfig, max_tokens: int, max_requests: int, device: int = 0,
                head_predicts_total: bool = False, precision: str = "auto", cls_last_layer: bool = False,
                residual16: bool | None = None) -> ElisConfig:
    """precision "auto" / residual16 None = the ABI defaults (elis.h ELIS_PREC_AUTO / ELIS_RESID_AUTO):
    fp16 operands + fp16 residual stream for head dim 64 encoders, bf16 + fp32 stream otherwise."""
    return ElisConfig(ABI_VERSION, cfg.vocab_size, cfg.max_position, cfg.type_vocab_size, cfg.num_layers, cfg.hidden,
                      cfg.num_heads, cfg.intermediate, cfg.ln_eps, cfg.pooling, cfg.head_layers, cfg.head_hidden,
                      int(head_predicts_total), int(max_tokens), int(max_requests), int(device), PRECISION[precision],
                      int(cls_last_layer), RESIDUAL[None if residual16 is None else bool(residual16)])


class Predictor:
    """Owner of one elis_predictor (device weights + workspaces)."""

    def __init__(self, cfg: inputs.EncoderConfig, flat_weights: np.ndarray, max_tokens: int, max_requests: int,
                 device: int = 0, head_predicts_total: bool = False, precision: str = "auto",
                 cls_last_layer: bool = False, residual16: bool | None = None):
        L = lib()
        self.cfg = cfg
        self.precision = precision
        self.residual16 = residual16
        self.c = make_config(cfg, max_tokens, max_requests, device, head_predicts_total, precision, cls_last_layer,
                             residual16)
        flat = np.ascontiguousarray(flat_weights, dtype=np.float32)
        need = L.elis_weight_count(ctypes.byref(self.c))
        if need != flat.size:
            raise ElisError(f"weight count {flat.size} != elis_weight_count {need}")
        h = _vp()
        check(L.elis_predictor_create(ctypes.byref(self.c), flat.ctypes.data, flat.size, ctypes.byref(h)),
              "elis_predictor_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().elis_predictor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path
    def predict_remaining(self, tokens, lengths, total_tokens: int, out_pred, out_slot=None, stream=None):
        n = int(lengths.shape[0])
        check(lib().elis_predict_remaining(self.h, _ptr(tokens), _ptr(lengths), n, int(total_tokens), _ptr(out_pred),
                                           _ptr(out_slot), _stream(stream)), "elis_predict_remaining")

    def predict_remaining_dev(self, tokens, lengths, dims, out_pred, out_slot=None, stream=None):
        """Shape-agnostic predict: n and total_tokens from the device tensor dims = [n, total]
        (graph-capturable; buffers sized for max_requests / max_tokens)."""
        check(lib().elis_predict_remaining_dev(self.h, _ptr(tokens), _ptr(lengths), _ptr(dims), _ptr(out_pred),
                                               _ptr(out_slot), _stream(stream)), "elis_predict_remaining_dev")

    def predict_remaining_dist(self, tokens, lengths, total_tokens: int, table, out_slot, stream=None):
        """This rank's due requests -> table[out_slot[i]] on EVERY attached rank (a collective)."""
        n = 0 if lengths is None else int(lengths.shape[0])
        check(lib().elis_predict_remaining_dist(self.h, _ptr(tokens), _ptr(lengths), n, int(total_tokens),
                                                _ptr(table), _ptr(out_slot), _stream(stream)),
              "elis_predict_remaining_dist")

    def iteration_table_host(self, tokens, lengths, slots, table, generated, batch_cap: int, out_ids,
                             out_count=None, stream=None):
        """Host due tokens / lengths / slots in, predict into the device table (all ranks when a
        transport is attached), select over the whole table, host ids out; synchronises."""
        n = int(lengths.shape[0])
        check(lib().elis_iteration_table_host(self.h, _ptr(tokens), _ptr(lengths), n, int(tokens.shape[0]),
                                              _ptr(slots), _ptr(table), _ptr(generated), int(generated.shape[0]),
                                              int(batch_cap), None, _ptr(out_ids), _ptr(out_count),
                                              _stream(stream)), "elis_iteration_table_host")

    def isrtf_select(self, pred, generated, batch_cap: int, out_ids, policy=POLICY_ISRTF, allow_preempt=True,
                     order=None, running=None, out_preempted=None, out_count=None, out_nan_count=None, stream=None,
                     windows_waited=None, boost_after=1, boost_amount=0.0, preempt_margin=0.0):
        pre = _preempt(policy, allow_preempt, order, running, out_preempted, out_count, out_nan_count,
                       windows_waited, boost_after, boost_amount, preempt_margin)
        check(lib().elis_isrtf_select(self.h, _ptr(pred), _ptr(generated), int(generated.shape[0]), int(batch_cap),
                                      ctypes.byref(pre), _ptr(out_ids), _stream(stream)), "elis_isrtf_select")

    def assign_nodes(self, node_load, n_new: int, out_node, stream=None):
        """Least-loaded node for each of n_new arriving jobs; node_load (device int32) updated."""
        check(lib().elis_assign_nodes(self.h, _ptr(node_load), int(node_load.shape[0]), int(n_new), _ptr(out_node),
                                      _stream(stream)), "elis_assign_nodes")

    def isrtf_select_nodes(self, pred, generated, node, num_nodes: int, batch_cap: int, out_ids, out_counts,
                           node_ready=None, policy=POLICY_ISRTF, allow_preempt=True, order=None, running=None,
                           out_preempted=None, out_nan_count=None, stream=None, windows_waited=None,
                           boost_after=1, boost_amount=0.0, preempt_margin=0.0):
        """Per-node batches: out_ids [num_nodes * batch_cap], out_counts [num_nodes] (device)."""
        pre = _preempt(policy, allow_preempt, order, running, out_preempted, None, out_nan_count,
                       windows_waited, boost_after, boost_amount, preempt_margin)
        check(lib().elis_isrtf_select_nodes(self.h, _ptr(pred), _ptr(generated), _ptr(node), _ptr(node_ready),
                                            int(generated.shape[0]), int(num_nodes), int(batch_cap),
                                            ctypes.byref(pre), _ptr(out_ids), _ptr(out_counts), _stream(stream)),
              "elis_isrtf_select_nodes")

    def dist_attach(self, rank: int, world: int, unique_id: bytes):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(lib().elis_dist_attach(self.h, rank, world, buf), "elis_dist_attach")

    def peer_export(self, rank: int, world: int) -> bytes:
        """Allocate this rank's peer region; return its 64-byte CUDA IPC handle."""
        buf = ctypes.create_string_buffer(64)
        check(lib().elis_peer_export(self.h, int(rank), int(world), buf), "elis_peer_export")
        return buf.raw

    def peer_attach(self, handles: list[bytes]):
        """Map every rank's region (handles in rank order, as all-gathered by the caller)."""
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * len(handles))
        check(lib().elis_peer_attach(self.h, buf), "elis_peer_attach")

    def isrtf_select_dist(self, pred, generated, global_offset: int, batch_cap: int, out_ids, policy=POLICY_ISRTF,
                          allow_preempt=True, order=None, running=None, out_preempted=None, out_count=None,
                          out_nan_count=None, stream=None):
        pre = _preempt(policy, allow_preempt, order, running, out_preempted, out_count, out_nan_count)
        check(lib().elis_isrtf_select_dist(self.h, _ptr(pred), _ptr(generated), int(generated.shape[0]),
                                           int(global_offset), int(batch_cap), ctypes.byref(pre), _ptr(out_ids),
                                           _stream(stream)), "elis_isrtf_select_dist")

    def iteration_host(self, tokens: np.ndarray, lengths: np.ndarray, generated: np.ndarray, batch_cap: int,
                       out_ids: np.ndarray, out_count: np.ndarray | None = None, out_pred: np.ndarray | None = None,
                       order: np.ndarray | None = None, running: np.ndarray | None = None, policy=POLICY_ISRTF,
                       allow_preempt=True, global_offset: int = -1, stream=None):
        """Host buffers in (numpy or pinned torch CPU tensors), ids out; synchronises.
        global_offset >= 0 selects globally over the attached NCCL communicator."""
        check(lib().elis_iteration_host(self.h, _ptr(tokens), _ptr(lengths), int(lengths.shape[0]),
                                        int(tokens.shape[0]), _ptr(generated), _ptr(order), _ptr(running),
                                        int(policy), int(allow_preempt), int(batch_cap), int(global_offset),
                                        _ptr(out_ids),
                                        _ptr(out_count), _ptr(out_pred), _stream(stream)), "elis_iteration_host")

    # ---- instrumentation
    def sync_status(self) -> int:
        return lib().elis_sync_status(self.h)

    def device_error_bits(self) -> int:
        return lib().elis_last_device_error_bits(self.h)

    def get_hidden(self, dst, stream=None):
        check(lib().elis_get_hidden(self.h, _ptr(dst), int(dst.numel()), _stream(stream)), "elis_get_hidden")

    def launch_count(self) -> int:
        return int(lib().elis_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        check(lib().elis_profile_enable(self.h, int(on)), "elis_profile_enable")

    def profile_read(self) -> dict:
        cap = 32
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_double * cap)()
        cnt = (ctypes.c_int64 * cap)()
        k = lib().elis_profile_read(self.h, names, ms, cnt, cap)
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(min(k, cap)) if cnt[i] > 0}


def peer_attach_local(predictors: list["Predictor"]):
    """Wire predictors of ONE process as ranks 0..world-1 of the peer-memory transport."""
    arr = (_vp * len(predictors))(*[P.h for P in predictors])
    check(lib().elis_peer_attach_local(arr, len(predictors)), "elis_peer_attach_local")


class Arena:
    """Owner of one elis_arena: the device-resident prompts and recent response tokens of an
    in-flight table (include/elis.h).  Device tensors in, argument marshalling only."""

    def __init__(self, max_slots: int, device: int = 0):
        h = _vp()
        check(lib().elis_arena_create(int(max_slots), int(device), ctypes.byref(h)), "elis_arena_create")
        self.h = h
        self.max_slots = max_slots

    def close(self):
        if self.h:
            lib().elis_arena_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_prompts(self, slots, tokens, lengths, stream=None):
        check(lib().elis_arena_set_prompts(self.h, _ptr(slots), _ptr(tokens), _ptr(lengths), int(slots.numel()),
                                           _stream(stream)), "elis_arena_set_prompts")

    def append(self, slots, tokens, counts, stream=None):
        check(lib().elis_arena_append(self.h, _ptr(slots), _ptr(tokens), _ptr(counts), int(slots.numel()),
                                      _stream(stream)), "elis_arena_append")

    def gather(self, slots, max_len: int, out_tokens, out_lengths, out_dims=None, stream=None):
        check(lib().elis_arena_gather(self.h, _ptr(slots), int(slots.numel()), int(max_len), _ptr(out_tokens),
                                      _ptr(out_lengths), _ptr(out_dims) if out_dims is not None else None,
                                      _stream(stream)), "elis_arena_gather")

    def sync_status(self, stream=None) -> int:
        return lib().elis_arena_sync_status(self.h, _stream(stream))


def cost_split(lengths: np.ndarray, world: int, cfg: inputs.EncoderConfig) -> np.ndarray:
    """elis_cost_split: world + 1 slice bounds of the requests at the quantiles of their encoder cost."""
    L = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.empty(world + 1, np.int32)
    check(lib().elis_cost_split(L.ctypes.data if L.size else None, int(L.size), int(world), cfg.num_layers,
                                cfg.hidden, cfg.intermediate, out.ctypes.data), "elis_cost_split")
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().elis_nccl_unique_id(buf), "elis_nccl_unique_id")
    return buf.raw


# ---- per-op entry points (tests / microbenchmarks)
def op_gemm(A, W, bias, out, epilogue: int, residual=None, stream=None):
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm(_ptr(A), _ptr(W), _ptr(bias), _ptr(residual), _ptr(out), M, N, K, epilogue,
                             _stream(stream)), "elis_op_gemm")


def op_gemm_ln(A, W, bias, resid_inout, gamma, beta, eps: float, outb, stream=None):
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm_ln(_ptr(A), _ptr(W), _ptr(bias), _ptr(resid_inout), _ptr(gamma), _ptr(beta), eps,
                                _ptr(outb), M, N, K, _stream(stream)), "elis_op_gemm_ln")


def op_quant_rows_e4m3(W, q, scale, post: float = 1.0, stream=None):
    rows, cols = W.shape
    check(lib().elis_op_quant_rows_e4m3(_ptr(W), rows, cols, _ptr(q), _ptr(scale), post, _stream(stream)),
          "elis_op_quant_rows_e4m3")


def op_gemm_f8(A, W, colscale, bias, out, epilogue: int, out_scale: float = 1.0, stream=None):
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm_f8(_ptr(A), _ptr(W), _ptr(colscale), _ptr(bias), _ptr(out), M, N, K, epilogue,
                                out_scale, _stream(stream)), "elis_op_gemm_f8")


def op_gemm_ln16(A, W, bias, resid_inout, gamma, beta, eps: float, global_stats: bool = False, stream=None):
    """fp16 A [M, K], W [N, K]; resid_inout fp16 [M, N] <- LN(A W^T + bias + resid_inout) in place."""
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm_ln16(_ptr(A), _ptr(W), _ptr(bias), _ptr(resid_inout), _ptr(gamma), _ptr(beta), eps,
                                  M, N, K, int(global_stats), _stream(stream)), "elis_op_gemm_ln16")


def op_gemm_ln_f8(A, W, colscale, bias, resid_inout, gamma, beta, eps: float, outb, out_scale: float, stream=None):
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm_ln_f8(_ptr(A), _ptr(W), _ptr(colscale), _ptr(bias), _ptr(resid_inout), _ptr(gamma),
                                   _ptr(beta), eps, _ptr(outb), out_scale, M, N, K, _stream(stream)),
          "elis_op_gemm_ln_f8")


def op_gemm_f16(A, W, bias, out, epilogue: int, head_major: bool = False, stream=None):
    M, K = A.shape
    N = W.shape[0]
    check(lib().elis_op_gemm_f16(_ptr(A), _ptr(W), _ptr(bias), _ptr(out), M, N, K, epilogue, int(head_major),
                                 _stream(stream)), "elis_op_gemm_f16")


def op_attention(qkv, lengths, hidden: int, num_heads: int, ctx, stream=None, f16: bool = False):
    fn = lib().elis_op_attention_f16 if f16 else lib().elis_op_attention
    check(fn(_ptr(qkv), _ptr(lengths), int(lengths.shape[0]), int(ctx.shape[0]), hidden, num_heads, _ptr(ctx),
             _stream(stream)), "elis_op_attention_f16" if f16 else "elis_op_attention")


def op_layernorm(u, gamma, beta, eps: float, out32, outb=None, stream=None):
    rows, H = u.shape
    check(lib().elis_op_layernorm(_ptr(u), _ptr(gamma), _ptr(beta), eps, rows, H, _ptr(out32), _ptr(outb),
                                  _stream(stream)), "elis_op_layernorm")


def op_fc_f32(X, W, b, Y, relu: bool, stream=None):
    n, K = X.shape
    N = W.shape[0]
    check(lib().elis_op_fc_f32(_ptr(X), _ptr(W), _ptr(b), _ptr(Y), n, N, K, int(relu), _stream(stream)),
          "elis_op_fc_f32")
