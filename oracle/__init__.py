"""CPU oracle for the gDist hot path -- test infrastructure only.

Imported by tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs as the checker or timed CPU baseline; never by the product
package.  Parity is pinned against golden vectors generated from the
reference itself (tests/golden/make_golden.py).
"""
