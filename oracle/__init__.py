"""CPU oracle for the skewstream hot path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports
it (tests/test_layout.py checks that).  Parity is pinned against the
reference itself through tests/golden/ (see port.py's header).
"""

from .port import *  # noqa: F401,F403
from . import port  # noqa: F401
