"""CPU oracle (test infrastructure only; see dinfer_oracle.py header)."""
from .dinfer_oracle import *  # noqa: F401,F403
