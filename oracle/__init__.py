"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_2204_03893_b200/) never imports it.
"""
from .oracle import (OracleCSR, assemble, assemble_tensor_contraction, basis, build, k_eval, dk_eval,
                     max_threads, pattern)
