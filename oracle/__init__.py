"""CPU oracle for the DynLP batch update -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
reference.  The product (``paper_2604_06596_b200``) never imports it and has
no CPU fallback.

* ``OracleEngine``: ctypes wrapper over oracle/dynlp_oracle.c, a plain-C
  restatement of ``engine.apply_batch`` (engine.py:328-413) and the kernel
  plugin functions of ``kernels/_csr.pyx``.
* ``load_reference()``: imports the unmodified reference compiled into
  ``oracle/_ref`` (see oracle/build.py), or the source tree when present.
"""

from .oracle import (  # noqa: F401
    OracleEngine,
    OracleReport,
    load_reference,
    orc_gauss_seidel_step,
    orc_jacobi_run,
    orc_jacobi_step,
    pairwise_sum,
)
