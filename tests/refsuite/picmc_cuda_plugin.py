"""pytest plugin: run the reference's OWN test suite with the cuda backend
selected, exactly as the two-line change in INTEGRATION.md §4 would select it
(`PICMC_BACKEND=cuda` in pkg/src/picmc/backends/__init__.py:18-50).

Loaded with `-p picmc_cuda_plugin` by tests/test_reference_suite_gpu.py; the
reference package is the unmodified install in baseline/_ref (made by
scripts/install_reference.sh).  At import time the plugin

* imports `picmc.backends` (with PICMC_BACKEND=compiled so the unmodified
  selector accepts the environment),
* adds "cuda" to its choices and makes `load_backend("cuda")` return
  `paper_2404_10270_b200.backend`,
* re-points the module-level kernels (`BACKEND`, `deposit_partials`,
  `gather`, `fused_move`, `fused_move_table`, `fused_move_aos`) at the cuda
  backend -- what `PICMC_BACKEND=cuda` does after the change.  Every caller in
  the reference (`mover.py:61,257`, `fields.py:71,230`, `layout_lab.py:182`)
  looks the kernels up on the module at call time, so the whole reference
  (mover_phase under its threaded Scheduler, deposit_charge, run_simulation,
  the acceptance criteria) now runs its hot kernels on the GPU.

With PICMC_CUDA_SUBSTITUTE=1 it additionally makes `load_backend("compiled")`
return the cuda backend, so pkg/tests/test_backends.py compares pure (NumPy)
against cuda bit for bit; the two tests there that assert backend NAMES
(`test_backend_selector`, `test_backend_names`) are deselected by the runner
in that mode.

Every cuda kernel call is counted; the counts are written to the file named
by PICMC_CUDA_CALLS at session end, as proof that the GPU path ran.
"""

import collections
import json
import os
import threading

os.environ["PICMC_BACKEND"] = "compiled"

import picmc  # noqa: E402
import picmc.backends as _pb  # noqa: E402

from paper_2404_10270_b200 import backend as _cuda  # noqa: E402

_calls = collections.Counter()
_lock = threading.Lock()


def _counted(name):
    fn = getattr(_cuda, name)

    def wrapper(*a, **k):
        with _lock:
            _calls[name] += 1
        return fn(*a, **k)

    wrapper.__name__ = name
    wrapper.__doc__ = fn.__doc__
    return wrapper


class _CountedCuda:
    BACKEND_NAME = _cuda.BACKEND_NAME
    deposit_partials = staticmethod(_counted("deposit_partials"))
    gather = staticmethod(_counted("gather"))
    fused_move = staticmethod(_counted("fused_move"))
    fused_move_table = staticmethod(_counted("fused_move_table"))
    fused_move_aos = staticmethod(_counted("fused_move_aos"))


_orig_load = _pb.load_backend
_substitute = os.environ.get("PICMC_CUDA_SUBSTITUTE") == "1"


def load_backend(name: str):
    if name == "cuda" or (_substitute and name == "compiled"):
        return _CountedCuda
    return _orig_load(name)


_pb._CHOICES = tuple(_pb._CHOICES) + ("cuda",)
_pb.load_backend = load_backend
_pb._impl = _CountedCuda
_pb.BACKEND = _CountedCuda.BACKEND_NAME
for _n in ("deposit_partials", "gather", "fused_move", "fused_move_table", "fused_move_aos"):
    setattr(_pb, _n, getattr(_CountedCuda, _n))


def pytest_report_header(config):
    return [f"picmc from {os.path.dirname(picmc.__file__)}; backend selected: {_pb.BACKEND}"
            + (" (compiled -> cuda substitution)" if _substitute else "")]


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("PICMC_CUDA_CALLS")
    if out:
        with open(out, "w") as f:
            json.dump({"calls": dict(_calls), "backend": _pb.BACKEND,
                       "picmc": os.path.dirname(picmc.__file__)}, f)
