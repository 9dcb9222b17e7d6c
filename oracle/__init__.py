"""CPU oracle for the ring3pc hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (ring3pc, /root/reference/pkg
/src/ring3pc) written as one all-party simulation, each function citing the
reference file:line it follows.  It is pinned against the golden vectors the
live reference produced (tests/golden/, tests/test_oracle.py).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import it, and only as the checker or the timed CPU baseline; the product
package never does.
"""
