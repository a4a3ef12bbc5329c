"""CPU oracle for the Pier hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline leg may import this package, and only as the checker (or as the
timed CPU baseline).  The product package ``paper_2511_17849_b200`` never
imports it and has no CPU fallback.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src/pier``).
"""
