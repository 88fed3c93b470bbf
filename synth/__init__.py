"""Seeded synthetic inputs (CSR graphs).  Holds none of the method's
arithmetic; shared by the oracle tests and the CUDA path."""
from .graphs import *  # noqa: F401,F403
from .graphs import CONFIGS, GraphConfig  # noqa: F401
