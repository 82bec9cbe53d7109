"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (see each module's
docstring): lens prescription texts, ray-batch laws, map-weight blobs and
the five workload configurations.  It may be imported by ``oracle/``,
``tests/``, ``bench.py`` and the product alike.
"""
from . import configs, lenses, rays  # noqa: F401
