"""CPU oracle for the EQP-IFT element path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference ``strom`` algorithm for the hot path
(element residual, distortion, reduced operator, Levenberg-Marquardt),
each function citing the reference file:line it follows.  It is pinned
against golden vectors produced by the unmodified reference
(``tests/golden/make_golden.py``; checked by ``tests/test_oracle_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / reference arm may import this package, and only as the checker
or the timed CPU baseline — never as the product path.
"""
