"""pytest plugin: run the REFERENCE's own test suite with its executor swapped
for the B200 path.

Loaded with ``-p ref_swap_plugin`` when pytest runs
``baseline/_ref/mlower_tests`` (the reference's tests, installed next to the
reference by tools/install_reference.sh).  Before any test module is imported
it rebinds ``mlower.runtime.execute`` -- and the copies other reference
modules bound at import time (``pipeline``, ``cli``) -- to a wrapper around
``paper_2301_13441_b200.api.execute``, which takes the reference's own
``KernelPlan`` and ``Tensor`` and returns a reference ``Tensor`` computed by
libcmlb.so on the GPU.  The reference's tests then exercise our executor
through their own harness (``helpers.compiled_vs_oracle``, batch invariance,
zero-row batches, optimized == unoptimized, the CLI's run/verify ...).

Plans the B200 path does not lower (e.g. hand-built single-kernel graphs with
integer inputs) raise ``UnresolvedKernel`` -- there is no CPU fallback -- and
are counted in ``unresolved``; the summary is written to $REF_SWAP_REPORT.
"""

from __future__ import annotations

import json
import os

STATS = {"gpu_executes": 0, "unresolved": 0, "unresolved_kernels": {}}


def pytest_configure(config):
    import mlower.cli
    import mlower.pipeline
    import mlower.runtime

    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.errors import UnresolvedKernel

    reference_execute = mlower.runtime.execute
    if os.environ.get("REF_SWAP_IMPL") == "binding":
        # the reference-side ctypes binding of INTEGRATION.md section 2
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration"))
        import mlower_b200
        bound = mlower_b200.make_execute(reference_execute)

        def execute(plan, x):
            out = bound(plan, x)
            STATS["gpu_executes"] = mlower_b200.STATS["b200"]
            STATS["interpreted"] = mlower_b200.STATS["interpreted"]
            return out
        _install(execute, reference_execute, config)
        return

    def execute(plan, x):
        try:
            out = api.execute(plan, x)
        except UnresolvedKernel as e:
            STATS["unresolved"] += 1
            key = str(e)[:120]
            STATS["unresolved_kernels"][key] = STATS["unresolved_kernels"].get(key, 0) + 1
            raise
        STATS["gpu_executes"] += 1
        return out

    _install(execute, reference_execute, config)


def _install(execute, reference_execute, config):
    import mlower.cli
    import mlower.pipeline
    import mlower.runtime
    execute.__wrapped__ = reference_execute
    for mod in (mlower.runtime, mlower.pipeline, mlower.cli):
        if getattr(mod, "execute", None) is reference_execute:
            mod.execute = execute
    config._ref_swap_execute = execute


def pytest_unconfigure(config):
    path = os.environ.get("REF_SWAP_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump(STATS, fh, indent=1)
