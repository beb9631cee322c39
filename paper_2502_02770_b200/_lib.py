"""ctypes binding of the C ABI in include/twilight.h (libtwilight.so).

This is the only place the shared library is loaded.  There is no fallback:
if the library is missing or fails to load, importing an op raises, and every
op checks that its tensors live on a CUDA device.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TW_LIB_PATH") or os.path.join(HERE, "_lib", "libtwilight.so")

TW_OK, TW_ERR_INVALID, TW_ERR_INDEX, TW_ERR_DEGENERATE, TW_ERR_CUDA = range(5)
TW_F32, TW_BF16 = 0, 1
TW_SELECT_FULL, TW_SELECT_QUEST, TW_SELECT_SINK_WINDOW, TW_SELECT_CHANNEL_PRUNED = 0, 1, 2, 3
TW_ESTIMATE_INT, TW_ESTIMATE_EXACT = 0, 1
PAGE_SIZE = 16
DEFAULT_CHUNK = 512
QBLOCK_BYTES = 1152


def qblock_bytes(bits: int) -> int:
    """TW_QBLOCK_BYTES_FOR: a (page, KV head) block of b-bit codes + 128 B of fp32 scale/zero."""
    return 256 * bits + 128
HEAD_DIM = 128
TOPP_BINS = 4096          # TW_TOPP_BINS
TOPP_MEMBER_CAP = 8192    # TW_TOPP_MEMBER_CAP

# every symbol include/twilight.h declares
EXPORTS = (
    "tw_version", "tw_max_work_items", "tw_quant_append", "tw_quant_build", "tw_quant_rows",
    "tw_quest_scores", "tw_select", "tw_estimate", "tw_topp", "tw_sparse_attention", "tw_sparse_attention_part",
    "tw_dense_attention", "tw_decode_step", "tw_estimate_tokens", "tw_topp_bisect", "tw_select_estimate_topp",
    "tw_select_estimate_topp_applies", "tw_vec_logits", "tw_vec_softmax", "tw_vec_readout_parts",
    "tw_vec_readout",
)


class DegenerateSelectionError(ValueError):
    """Renormalization requested for a selection carrying no attention mass
    (reference: attention.py:30-31)."""


class TwPagedKV(ctypes.Structure):
    _fields_ = [
        ("num_seqs", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("group_size", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("max_pages", ctypes.c_int32), ("num_phys_pages", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("bits", ctypes.c_int32),
        ("k_cache", ctypes.c_void_p), ("v_cache", ctypes.c_void_p), ("kq", ctypes.c_void_p),
        ("kmeta", ctypes.c_void_p), ("kabsmax", ctypes.c_void_p), ("page_table", ctypes.c_void_p),
        ("seq_lens", ctypes.c_void_p),
    ]


class TwDecodeParams(ctypes.Structure):
    _fields_ = [
        ("selector", ctypes.c_int32), ("budget_pages", ctypes.c_int32), ("p", ctypes.c_double),
        ("chunk_tokens", ctypes.c_int32), ("renormalize", ctypes.c_int32), ("sink", ctypes.c_int32),
        ("window", ctypes.c_int32), ("top_channels", ctypes.c_int32), ("budget_tokens", ctypes.c_int32),
        ("channels_fixed", ctypes.c_int32), ("estimator", ctypes.c_int32),
    ]


class TwDecodeBuffers(ctypes.Structure):
    _fields_ = [
        ("page_scores", ctypes.c_void_p), ("cand_pages", ctypes.c_void_p), ("cand_count", ctypes.c_void_p),
        ("logits", ctypes.c_void_p), ("head_max", ctypes.c_void_p), ("head_thr", ctypes.c_void_p),
        ("head_stats", ctypes.c_void_p), ("final_idx", ctypes.c_void_p), ("final_count", ctypes.c_void_p),
        ("unit_items", ctypes.c_void_p), ("work_items", ctypes.c_void_p), ("counters", ctypes.c_void_p),
        ("partials", ctypes.c_void_p), ("head_page_bits", ctypes.c_void_p), ("sel_bits", ctypes.c_void_p),
        ("tok_mask", ctypes.c_void_p), ("chan_ids", ctypes.c_void_p), ("topp_done", ctypes.c_void_p), ("band_idx", ctypes.c_void_p), ("band_scores", ctypes.c_void_p),
        ("max_items", ctypes.c_int64),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libtwilight.so (raises if absent -- there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2502_02770_b200.build` "
            "(the Twilight path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I32 = ctypes.c_int32
    sig = {
        "tw_version": ([], I32),
        "tw_max_work_items": ([P, I32], ctypes.c_int64),
        "tw_quant_append": ([P, P, P, P, P], ctypes.c_int),
        "tw_quant_build": ([P, P], ctypes.c_int),
        "tw_quant_rows": ([P, I32, I32, I32, I32, P, P, P, P], ctypes.c_int),
        "tw_quest_scores": ([P, P, P, P], ctypes.c_int),
        "tw_select": ([P, P, P, P, P], ctypes.c_int),
        "tw_estimate": ([P, P, P, P, P], ctypes.c_int),
        "tw_topp": ([P, P, P, P], ctypes.c_int),
        "tw_sparse_attention": ([P, P, P, P, P, P], ctypes.c_int),
        "tw_sparse_attention_part": ([P, P, P, P, P, I32, P], ctypes.c_int),
        "tw_dense_attention": ([P, P, P, P, P], ctypes.c_int),
        "tw_decode_step": ([P, P, P, P, P, P, P, P, P], ctypes.c_int),
        "tw_estimate_tokens": ([P, I32, I32, P, P, I32, P, P, P], ctypes.c_int),
        "tw_topp_bisect": ([P, I32, I32, ctypes.c_double, ctypes.c_double, I32, P, P, P, P], ctypes.c_int),
        "tw_select_estimate_topp": ([P, P, P, P, P, P, P, P], ctypes.c_int),
        "tw_select_estimate_topp_applies": ([P, P, P], I32),
        "tw_vec_logits": ([P, P, ctypes.c_int64, I32, I32, P, P], ctypes.c_int),
        "tw_vec_softmax": ([P, ctypes.c_int64, P, P, P], ctypes.c_int),
        "tw_vec_readout_parts": ([], I32),
        "tw_vec_readout": ([P, I32, P, I32, ctypes.c_int64, I32, P, ctypes.c_int64, I32, P, P, P, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int, what: str) -> None:
    """Map a tw_status to the reference's exception types."""
    if status == TW_OK:
        return
    if status == TW_ERR_INVALID:
        raise ValueError(f"{what}: invalid argument")
    if status == TW_ERR_INDEX:
        raise IndexError(f"{what}: index out of range")
    if status == TW_ERR_DEGENERATE:
        raise DegenerateSelectionError(f"{what}: degenerate selection")
    raise RuntimeError(f"{what}: CUDA error {status}")


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must live on a CUDA device (the Twilight path has no CPU fallback)")
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return TW_BF16
    if dt == torch.float32:
        return TW_F32
    raise ValueError(f"dtype {dt} not supported on the B200 path (bf16 or float32)")
