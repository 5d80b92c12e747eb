"""fp64 CPU oracle for ARA with secondary uncertainty (arXiv 1310.2274).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA product path
(``paper_1310_2274_b200``) and neither imports the other.

- ``ara_oracle.c`` : Algorithm 1, section 3 sampler,
  financial terms, special functions, Philox (reading G4).
- ``core.py``      : ctypes wrapper around ``liboracle.so``.
- ``measures.py``  : PML / TVaR from a YLT by a full sort (SPEC
  conventions S:345-387, readings G13b/G16/G17).
"""
from .core import *  # noqa: F401,F403
from .measures import *  # noqa: F401,F403
