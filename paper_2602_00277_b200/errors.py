"""Error taxonomy of the FTAR data plane (drop-in for ftdp.errors).

Same two severities and the same reason tags as the reference
(pkg/src/ftdp/errors.py:11-22, classes :25-59), so callers written against
the reference catch the same exceptions.  The C-ABI reports integer status
codes; ``from_status`` maps them 1:1 onto these classes.
"""

from __future__ import annotations

TIMEOUT = "timeout"
PEER_RESET = "peer_reset"
PEER_DOWN = "peer_down"

PROTOCOL_VIOLATION = "protocol_violation"
NUMERICAL = "numerical"
INTERNAL_INVARIANT = "internal_invariant"

RECOVERABLE_REASONS = frozenset({TIMEOUT, PEER_RESET, PEER_DOWN})
FATAL_REASONS = frozenset({PROTOCOL_VIOLATION, NUMERICAL, INTERNAL_INVARIANT})


class FtdpError(Exception):
    """Base class; ``reason`` is one tag of the fixed taxonomy."""

    severity = "fatal"

    def __init__(self, reason: str, detail: str = ""):
        self.reason = reason
        self.detail = detail
        super().__init__(f"{reason}: {detail}" if detail else reason)


class Recoverable(FtdpError):
    """Lost/slow peer: the caller regroups through the quorum and retries."""

    severity = "recoverable"

    def __init__(self, reason: str, detail: str = ""):
        if reason not in RECOVERABLE_REASONS:
            raise ValueError(f"not a recoverable reason: {reason}")
        super().__init__(reason, detail)


class Fatal(FtdpError):
    """Protocol garbage, poisoned numerics or a broken invariant."""

    severity = "fatal"

    def __init__(self, reason: str, detail: str = ""):
        if reason not in FATAL_REASONS:
            raise ValueError(f"not a fatal reason: {reason}")
        super().__init__(reason, detail)


class ConfigError(Exception):
    """Bad runtime configuration."""


class InvariantViolation(Exception):
    """A checked run invariant failed."""


# C-ABI status codes (include/ftar_b200.h)
ST_OK = 0
ST_TIMEOUT = 1
ST_PEER_RESET = 2
ST_PEER_DOWN = 3
ST_PROTOCOL = 4
ST_NUMERICAL = 5
ST_INVARIANT = 6
ST_ABORTED = 7
ST_INJECTED = 8
ST_UNAVAILABLE = 9
ST_CUDA = 10
ST_PENDING = 255


def from_status(code: int, detail: str = "") -> FtdpError | None:
    """Exception for a non-zero C-ABI status (None for ST_OK)."""
    if code == ST_OK:
        return None
    if code == ST_TIMEOUT:
        return Recoverable(TIMEOUT, detail or "peer flag never arrived before the device deadline")
    if code == ST_ABORTED:
        return Recoverable(TIMEOUT, detail or "no progress within per_chunk_timeout_s; collective aborted")
    if code == ST_PEER_RESET:
        return Recoverable(PEER_RESET, detail or "peer aborted the collective")
    if code == ST_PEER_DOWN:
        return Recoverable(PEER_DOWN, detail or "peer unreachable")
    if code == ST_INJECTED:
        return Recoverable(PEER_DOWN, detail or "member stopped by fault injection")
    if code == ST_PROTOCOL:
        return Fatal(PROTOCOL_VIOLATION, detail or "peer announced a different call")
    if code == ST_NUMERICAL:
        return Fatal(NUMERICAL, detail or "non-finite values in reduction payload")
    if code == ST_INVARIANT:
        return Fatal(INTERNAL_INVARIANT, detail)
    if code == ST_CUDA:
        return Fatal(INTERNAL_INVARIANT, detail or "CUDA error")
    return Fatal(INTERNAL_INVARIANT, f"unknown status {code}: {detail}")
