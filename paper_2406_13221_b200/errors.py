"""Exceptions of the evaluator protocol.

``NeedsBootstrap`` mirrors ``helr.hesim.NeedsBootstrap`` (hesim.py:37-38):
raised by an evaluator when an operation would leave fewer than
``log_delta`` bits of modulus (hesim.py:136-142), caught by the training
driver, which refreshes W / V and re-runs the iteration
(enctrain.py:386-393).  Any evaluator plugged into ``train_encrypted`` via
``ctx=`` signals a level shortfall with this class (or a subclass).
"""

from __future__ import annotations

__all__ = ["NeedsBootstrap"]


class NeedsBootstrap(Exception):
    """Level shortfall: the operation needs a refresh first."""
