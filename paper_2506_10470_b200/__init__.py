"""B200-native TD-Pipe hot path (arxiv 2506.10470).

The product is the C-ABI shared library ``libtdpipe.so`` (include/tdpipe.h),
hand-written CUDA for sm_100a plus a C++ controller; ``tdpipe`` is a thin
ctypes binding with the same names.  There is no CPU fallback.
"""
from .tdpipe import (TD_BATCH_DECODE, TD_BATCH_PREFILL, TD_EXEC_CUDA, TD_EXEC_NULL, TD_POLICY_PPSB_ALT,
                     TD_POLICY_PPHB,
                     TD_POLICY_PPSB_PRIO, TD_POLICY_TDPIPE, TDError, TDPipe, default_options, lib, td_nccl_ids)

__all__ = ["TDPipe", "TDError", "lib", "default_options", "td_nccl_ids", "TD_EXEC_CUDA", "TD_EXEC_NULL",
           "TD_POLICY_TDPIPE", "TD_POLICY_PPSB_PRIO", "TD_POLICY_PPSB_ALT", "TD_POLICY_PPHB", "TD_BATCH_PREFILL",
           "TD_BATCH_DECODE"]
