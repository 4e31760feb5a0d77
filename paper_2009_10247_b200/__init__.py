"""B200-native (sm_100a) least-model and stable-model engine for propositional logic
programs, after "sparse matrix representation of logic programs" (arXiv 2009.10247).

The hot path -- the thresholded sparse mat-vec fixpoint v_{k+1} = θ(M_P v_k), its
frontier variant and the batched stable-model search -- runs in hand-written CUDA
kernels behind the C ABI of include/lp.h (liblp_b200.so).  This package is the thin
Python binding of that ABI; PyTorch is used only for device memory and streams.
"""
from .lp import (LIB_PATH, LPError, Program, bits_words, library, lp_free, lp_guess_model,
                 lp_info, lp_least_model, lp_load, lp_negated_atoms, lp_stable_matrix,
                 lp_shard_combine, lp_stable_models, lp_stable_search, pack_mask, unpack_bits)

__all__ = ["LIB_PATH", "LPError", "Program", "bits_words", "library", "lp_free", "lp_guess_model",
           "lp_info", "lp_least_model", "lp_load", "lp_negated_atoms", "lp_stable_matrix",
           "lp_shard_combine", "lp_stable_models", "lp_stable_search", "pack_mask", "unpack_bits"]
