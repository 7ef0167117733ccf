"""CPU oracle for the operator-representation inference path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2301_13441_b200`` imports,
links or executes anything under ``oracle/``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs use it, and only as the checker or the timed CPU baseline,
never as a code path of the product.

Two restatements of the reference ``mlower.runtime.execute`` semantics live
here (the reference itself is pure Python and cannot travel to the GPU box):

* :mod:`oracle.semantics` -- numpy, kernel by kernel, using the same numpy
  reductions the reference kernels use (``pkg/src/mlower/kernels.py``), so the
  summation order and rounding are identical by construction;
* ``oracle/cml_oracle.c`` (``oracle/liboracle.so``) -- multi-threaded C for
  full-size inputs and the CPU baseline, replaying numpy's reduction order
  explicitly; it is checked against :mod:`oracle.semantics` in the CPU suite.

Parity is pinned: ``tests/test_oracle_golden.py`` checks both against golden
vectors produced by running the reference itself (``tools/make_golden.py``,
outputs in ``tests/golden/``).
"""
