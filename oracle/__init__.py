"""Test-only CPU oracle for the Lloyd hot path (see lloyd_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package never imports this.
"""
from .lloyd_oracle import *  # noqa: F401,F403
from . import lloyd_oracle  # noqa: F401
from . import kernel_oracle  # noqa: F401,E402
