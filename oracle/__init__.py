"""CPU oracle for the approximate-activation training step (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline -- never as the product path.  The product
(``paper_1901_07988_b200``) never imports it and has no CPU fallback.

Pinned against the reference: ``tests/golden/*.npz`` are produced by
``tests/golden/make_golden.py`` which imports the unmodified reference
``qtape`` from ``/root/reference/pkg/src``; ``tests/test_oracle_golden.py``
checks this restatement against those fixtures (bit-exact for codes and the
fixed-order forward, tolerance for BLAS-ordered backward sums).
"""

from .qtape_oracle import *  # noqa: F401,F403
