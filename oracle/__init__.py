"""Test-infrastructure oracle (see cp_oracle.py header).  Never imported by the product path."""
from .cp_oracle import *  # noqa: F401,F403
