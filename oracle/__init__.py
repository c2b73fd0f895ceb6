"""CPU oracle for the VP-FV stage hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import anything from this package.  The product
package (``paper_2410_12155_b200``) never imports, links or executes it: the
product path is the sm_100a CUDA library and fails loudly without it.

Contents
--------
``vpfv_oracle``   numpy restatement of the reference algorithm (each function
                  cites the /root/reference file:line it restates).
``stage_ref.c``   plain-C restatement of the fused stage kernels and the fold-
                  tree moment (OpenMP over the outermost dimension, compiled
                  without FMA contraction so it is bitwise equal to the
                  reference's numba kernels); used as the multi-core CPU
                  baseline.
``cbackend``      ctypes loader for the compiled C restatement.

Parity is pinned: ``tests/golden/make_golden.py`` imports the real reference
(only possible in the build container, where /root/reference exists) and
writes the fixtures under ``tests/golden/`` that ``tests/test_oracle.py``
checks this oracle against, bit for bit where the reference is bitwise
reproducible.
"""
