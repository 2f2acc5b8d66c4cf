"""Test infrastructure: the CPU checkers for the Merge Path hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline -- never as the thing measured or shipped.

  oracle.bindings.port()  -> liboracle.so, the C restatement (mp_oracle.c)
  oracle.bindings.ref()   -> _ref/libmergepath_ref.so, the unmodified
                             reference library behind ref_shim.cpp
"""
