"""Import the read-only reference (`mlpsort`) — TEST INFRASTRUCTURE ONLY.

Only available in the build container (``/root/reference`` does not exist on
the GPU box).  Used by ``oracle/make_goldens.py`` to produce the committed
fixtures and by ``bench.py --impl reference`` when the reference is present.
"""

from __future__ import annotations

import os
import sys

REF_SRC = os.environ.get("AMS_REFERENCE_SRC", "/root/reference/pkg/src")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "mlpsort"))


def load():
    """Return the ``mlpsort`` package (imported without writing bytecode
    into the read-only tree)."""
    if not available():
        raise ImportError(f"reference not found at {REF_SRC}")
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mlpsort  # noqa: F401
    import mlpsort.ams  # noqa: F401
    import mlpsort.bench  # noqa: F401
    return sys.modules["mlpsort"]
