"""B200-native check-belief propagation (CBP) decoding of QC-LDPC codes.

Guan & Liang, "Check-Belief Propagation Decoding of LDPC Codes" (arXiv
2305.05286).  The hot path runs in sm_100a kernels behind the C ABI of
include/cbp.h (libcbp.so); this package is the thin Python binding plus the
multi-GPU counter reduction (dist.py).
"""
from .cbp import (ALPHA_DEFAULT, CBP_ALG_FBP, CBP_ALG_LBP, CBP_ALG_LOG_TANH, CBP_ALG_MIN_SUM, CBP_LLR_INT8, CBP_TX_ZERO, CBP_STOP_BELIEF_M, CBP_STOP_BELIEF_N, CBP_STOP_NONE, CBP_STOP_SYNDROME, COUNT_NAMES, CbpError,
                  Code, construct_base, lib, unpack_bits)

__all__ = ["ALPHA_DEFAULT", "CBP_LLR_INT8", "CBP_TX_ZERO", "CBP_ALG_LOG_TANH", "CBP_ALG_MIN_SUM", "CBP_ALG_LBP", "CBP_ALG_FBP", "Code", "construct_base", "lib", "unpack_bits", "CbpError", "COUNT_NAMES", "CBP_STOP_BELIEF_M",
           "CBP_STOP_BELIEF_N", "CBP_STOP_SYNDROME", "CBP_STOP_NONE"]
