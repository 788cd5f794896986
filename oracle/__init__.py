"""CPU oracle for the my_dgemm path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package, and only as the checker or the timed CPU baseline.  The product
package (paper_1609_00076_b200) never imports it; see oracle/oracle.c for the
restated algorithm and its reference citations.
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
