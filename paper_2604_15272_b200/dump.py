"""tile_dump support for run_concrete (interp.py:132,210-211)."""
from __future__ import annotations

from .errors import UnsupportedOpError


def run_with_dump(concrete, inputs, dtype, tile_dump, device=None):
    raise UnsupportedOpError("tile_dump needs the dump-mode kernel variant (not built yet)")
