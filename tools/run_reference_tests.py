"""Run the reference's own test files against the B200 drop-in by import aliasing.

    python tools/run_reference_tests.py <reference tests dir> [pytest args...]

``import trihalo`` (and its submodules) resolves to paper_2504_15814_b200: the
package-level names, geometry, schemes, errors and harness are the drop-in's own
modules; taylor / csr / linear / linalg are assembled from the drop-in's operator
cache, CSR I/O and construction modules.  ``trihalo.cli`` is a stub (the CLI is out
of scope).  The reference test files are NOT part of this repository: the caller
points at a copy (for a GPU box, a git-ignored copy under baseline/_ref/, next to the
reference install that travels there).
"""

from __future__ import annotations

import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def install_aliases() -> None:
    import paper_2504_15814_b200 as th
    from paper_2504_15814_b200 import construction, csrio, errors, geometry, harness, operators, schemes

    def module(name, *sources, **extra):
        m = types.ModuleType(name)
        for src in sources:
            for k in dir(src):
                if not k.startswith("__"):
                    setattr(m, k, getattr(src, k))
        for k, v in extra.items():
            setattr(m, k, v)
        return m

    taylor = module("trihalo.taylor", construction, operators)
    csr = module("trihalo.csr", operators, csrio)
    linear = module("trihalo.linear", construction)
    linalg = module("trihalo.linalg", errors, construction)

    def _no_cli(*a, **k):
        raise NotImplementedError("the trihalo CLI is outside the B200 hot-path scope")

    cli = module("trihalo.cli", main=_no_cli)
    pkg = module("trihalo", th, geometry=geometry, schemes=schemes, errors=errors, harness=harness, taylor=taylor,
                 csr=csr, linear=linear, linalg=linalg, cli=cli)
    pkg.__path__ = []
    sys.modules.update({"trihalo": pkg, "trihalo.geometry": geometry, "trihalo.schemes": schemes,
                        "trihalo.errors": errors, "trihalo.harness": harness, "trihalo.taylor": taylor,
                        "trihalo.csr": csr, "trihalo.linear": linear, "trihalo.linalg": linalg,
                        "trihalo.cli": cli})


def main(argv) -> int:
    import pytest

    install_aliases()
    tests = os.path.abspath(argv[0])
    sys.path.insert(0, tests)  # the reference's conftest helpers (from conftest import ...)
    args = [a if a.startswith("-") or not (a.endswith(".py") or "::" in a) else os.path.join(tests, a)
            for a in argv[1:]]
    if not any(a.endswith(".py") or "::" in a for a in args):
        args.append(tests)
    os.chdir(tests)  # the repository's own pytest.ini (testpaths = tests) must not apply
    return pytest.main(["-p", "no:cacheprovider", "-c", os.devnull, "--rootdir", tests, *args])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
