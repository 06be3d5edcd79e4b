"""Locate the reference's strategy/rewrite API (`stratir`).

The backend is a drop-in *below* the reference's rewriting stack: schedules are
built with the reference's own rules, traversals and normal forms, and the
dispatch reads terms with its `ir`/`typecheck` modules.  Those modules are the
unmodified reference package, installed (git-ignored) into `baseline/_ref` by
`__graft_entry__.build()` with
`pip install --no-index --no-build-isolation --target baseline/_ref <copy of
/root/reference/pkg>`.  `baseline/_ref` travels to the GPU box with the repo
snapshot; `/root/reference` itself is never read at run time by the product.

Nothing here evaluates programs: the reference interpreter (`stratir.interp`)
is only used by tests and by bench.py's CPU-baseline leg.
"""

from __future__ import annotations

import importlib
import os
import sys

REPO_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(REPO_ROOT, "baseline", "_ref")


def _ensure_path() -> None:
    if os.path.isdir(os.path.join(REF_INSTALL, "stratir")) and REF_INSTALL not in sys.path:
        sys.path.insert(0, REF_INSTALL)


def stratir():
    """Import and return the reference package's modules as a namespace."""
    _ensure_path()
    try:
        mods = {m: importlib.import_module(f"stratir.{m}")
                for m in ("ir", "typecheck", "rules", "strategy", "traversals",
                          "normal_forms", "interp")}
    except ImportError as e:  # pragma: no cover - environment problem
        raise ImportError(
            "the reference strategy API (stratir) is not installed; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` to install it "
            f"into {REF_INSTALL}") from e

    class _NS:
        pass

    ns = _NS()
    for k, v in mods.items():
        setattr(ns, k, v)
    return ns


_S = None


def S():
    global _S
    if _S is None:
        _S = stratir()
    return _S
