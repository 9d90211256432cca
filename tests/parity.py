"""The fast-mode tolerance checker lives in oracle/parity.py (test
infrastructure shared with __graft_entry__.smoke())."""

from oracle.parity import MAX_RTOL, MPV_RTOL, NEAR_ZERO, check_fast  # noqa: F401
