"""CPU oracle for the Dummy Forcing attention hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline.  The product path
(``paper_2601_20499_b200``) never imports it and has no CPU fallback.

The restatement follows /root/reference/pkg/src/dummy_forcing (numpy); each
function cites the file:line it restates.  It is pinned against golden vectors
generated from the reference itself by ``oracle/gen_golden.py`` (committed
under ``tests/golden/``) -- see tests/test_oracle_golden.py.
"""
