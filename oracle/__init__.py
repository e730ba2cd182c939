"""ORACLE -- test infrastructure only (see oracle/oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path never does.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import (apply_gate, simulate, norm, init_basis, embed_dense,  # noqa: F401
                     kron_embed_adjacent, circuit_matrix, tensordot_apply,
                     compress, fused_gates, build_oracle, set_threads, max_threads,
                     OracleError, init_tokens, project, probabilities, dm_apply_kraus, dm_vec,
                     reduced_dm, kraus_sample_step, reversible_image)
