"""CPU oracle for the RSR hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference algorithm of every function on
the hot path (sampling -> dominance classification -> Phi -> boundary search
-> reference-set maintenance -> P-hat / c.o.v. accumulation).  Each function
cites the reference file:line it follows (paths relative to the reference
package root ``pkg/src/rsr/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it, and only as the checker or as the
timed CPU baseline.  The product package ``paper_2604_17066_b200`` never
imports it: the device path fails loudly when its CUDA library is missing.

Parity pin: the restatement is checked against golden vectors generated from
the reference package itself (``tests/golden/make_golden.py``, run in the
build container where the reference is importable) and against numpy's own
``np.random.Philox`` for the Philox4x64-10 stream (numpy 2.3.5 is the
reference's arithmetic dependency; ``pkg/pyproject.toml:9``).
"""

from .philox import philox4x64_blocks, random_raw, uniform_field  # noqa: F401
from .core import *  # noqa: F401,F403
