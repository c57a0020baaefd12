"""Locate the reference scheduler package ``epdsim``.

The executor drops in *under* the reference's own stage-level scheduler and trace
replayer, so ``epdsim`` is a runtime dependency of the host side.  It is looked up
on ``sys.path`` first, then in ``$EPDSIM_PATH``, then in the repo's offline install
``baseline/_ref`` (``pip install --target baseline/_ref`` of the reference package,
see DESIGN.md).  Missing it is an error, never a silent fallback.
"""

from __future__ import annotations

import importlib
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_epdsim():
    try:
        return importlib.import_module("epdsim")
    except ImportError:
        pass
    for cand in (os.environ.get("EPDSIM_PATH"), os.path.join(_REPO, "baseline", "_ref")):
        if cand and os.path.isdir(os.path.join(cand, "epdsim")):
            if cand not in sys.path:
                sys.path.append(cand)
            return importlib.import_module("epdsim")
    raise ImportError("epdsim (the reference scheduler) not found: install it with "
                      "`pip install --no-deps --target baseline/_ref <reference pkg>` "
                      "or set EPDSIM_PATH")


E = load_epdsim()
import epdsim.cluster as C  # noqa: E402
import epdsim.engine as EN  # noqa: E402
import epdsim.migration as MG  # noqa: E402
import epdsim.model_cost as MC  # noqa: E402
