#!/usr/bin/env python
"""Stage the reference's own test suite to run against this package.

Copies /root/reference/pkg/tests into ``.refsuite/tests`` (git-ignored; the
files are the reference's, so they are never committed) next to a
``dimscan`` shim package whose modules re-export this package's
(``dimscan.bench`` -> ``synthetic``, the others by the same name), so
``import dimscan`` in those tests binds the B200 implementation.  Run the
staged suite on a GPU box with

    python -m pytest .refsuite/tests -q -p no:cacheprovider

(tests/test_reference_suite.py does that when ``.refsuite`` exists) and
delete ``.refsuite`` afterwards.
"""
from __future__ import annotations

import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/pkg/tests")
MODULES = {"bench": "synthetic", "estimators": "estimators", "index": "index",
           "kernels": "kernels", "layout": "layout", "pruning": "pruning", "search": "search",
           "storage": "storage", "cli": "cli"}


def main():
    dst = ROOT / ".refsuite"
    if dst.exists():
        shutil.rmtree(dst)
    (dst / "dimscan").mkdir(parents=True)
    shutil.copytree(SRC, dst / "tests")
    # submodules first, then the package namespace (as dimscan/__init__.py
    # does): a later `import dimscan.search` must not rebind `dimscan.search`
    (dst / "dimscan" / "__init__.py").write_text(
        "".join(f"from . import {name}  # noqa: F401\n" for name in MODULES) +
        "from paper_2503_04422_b200 import *  # noqa: F401,F403\n"
        "from paper_2503_04422_b200 import __version__  # noqa: F401\n")
    for name, ours in MODULES.items():
        (dst / "dimscan" / f"{name}.py").write_text(
            f"from paper_2503_04422_b200.{ours} import *  # noqa: F401,F403\n"
            f"from paper_2503_04422_b200 import {ours} as _m\n"
            "globals().update({k: v for k, v in vars(_m).items() if not k.startswith('__')})\n")
    (dst / "conftest.py").write_text(
        "import sys\nfrom pathlib import Path\n"
        "HERE = Path(__file__).resolve().parent\n"
        "sys.path.insert(0, str(HERE))\nsys.path.insert(0, str(HERE.parent))\n")
    print(f"staged {sum(1 for _ in (dst / 'tests').glob('test_*.py'))} reference test files "
          f"into {dst}")


if __name__ == "__main__":
    sys.exit(main())
