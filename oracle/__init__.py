"""CPU oracle for the ZoomR select + sparse-decode hot path (arXiv 2604.10898).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2604_10898_b200`` never imports it, and
the two share no code: the oracle is plain C (``zoomr_oracle.c``) in fp64 plus
this ctypes marshalling layer, which holds none of the method's arithmetic.
"""
from .oracle import *  # noqa: F401,F403
