"""TEST INFRASTRUCTURE ONLY: CPU oracles for the DELTA path.

* `oracle.ref`   — ctypes binding to the UNMODIFIED reference simulator built
  from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
* `oracle.delta_oracle` — a pure-Python restatement of the reference
  algorithm (engine/policy/state), each function citing the reference
  file:line it follows.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package; the product path (paper_2203_15980_b200) never does.
"""
