"""`import h2ulv` -> this package: the switch a user of the reference makes.

`install()` registers the package and its modules under the reference's
module names (pkg/src/h2ulv/__init__.py:1-14), so code written against
`h2ulv` — including the reference's own test-suite — runs unchanged on the
GPU path:

    from paper_2502_02395_b200 import h2ulv_compat
    h2ulv_compat.install()
    from h2ulv.ulv_factor import factorize          # the GPU factorization

Modules of the reference that are outside this build's hot path (the dense
oracle, the communication simulator, the CLI) are
not provided by the package.  `install(extra_dir=...)` loads them from a
directory holding the reference's own files, as submodules of the alias, so
their relative imports (`from . import kernels`) bind to this package's
modules.  That is test infrastructure (oracle/_ref, see
oracle/make_ref_suite.py): the product path never uses it.
"""

import importlib.util
import os
import sys

PROVIDED = ("dense_core", "errors", "geometry", "h2_build", "kernels", "storage", "ulv_factor", "ulv_solve")


def install(extra_dir=None, extra=("oracle", "comm_sim", "cli")):
    import paper_2502_02395_b200 as pkg

    sys.modules["h2ulv"] = pkg
    for name in PROVIDED:
        mod = importlib.import_module(f"paper_2502_02395_b200.{name}")
        sys.modules[f"h2ulv.{name}"] = mod
    if extra_dir is None:
        return pkg
    for name in extra:
        path = os.path.join(extra_dir, f"{name}.py")
        full = f"h2ulv.{name}"
        if full in sys.modules or not os.path.exists(path):
            continue
        spec = importlib.util.spec_from_file_location(full, path)
        mod = importlib.util.module_from_spec(spec)
        mod.__package__ = "h2ulv"
        sys.modules[full] = mod
        spec.loader.exec_module(mod)
        setattr(pkg, name, mod)
    return pkg
