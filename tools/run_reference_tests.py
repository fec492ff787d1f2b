"""Run the REFERENCE's own test suite (pkg/tests, copied into
baseline/_ref/halftile_tests by tools/install_reference.sh) against this
repo's drop-in: ``import halftile`` resolves to paper_1811_09736_b200 (the
B200 kernels), while the reference's exact oracle (``halftile.oracle``) and
anything the drop-in does not re-implement (the simulator's binary16 scalar
type, the fragment internals) come from the installed reference -- they are
the checker, not the thing under test.

usage (GPU box): python tools/run_reference_tests.py [pytest args...]

Deselected: test_engine.py and test_half.py (the simulator's tile engine and
binary16 library -- not the hot path) and the asserts on
the simulator's MMA / cycle counters (-k filters below), which count 16x16
warp MMAs of a 2018 GPU model rather than results.
"""

import importlib
import importlib.abc
import importlib.util
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
TESTS = REF / "halftile_tests"

OURS = "paper_1811_09736_b200"
# submodules taken from the reference (the checker side)
FROM_REF = {"oracle"}


def _load_reference():
    """Import the installed reference under the private name _ref_halftile."""
    saved = {k: v for k, v in sys.modules.items() if k == "halftile" or k.startswith("halftile.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, str(REF))
    try:
        ref = importlib.import_module("halftile")
        for f in sorted((REF / "halftile").glob("*.py")):
            if f.stem != "__init__":
                importlib.import_module(f"halftile.{f.stem}")
        mods = {k: v for k, v in sys.modules.items() if k == "halftile" or k.startswith("halftile.")}
    finally:
        sys.path.remove(str(REF))
        for k in list(sys.modules):
            if k == "halftile" or k.startswith("halftile."):
                del sys.modules[k]
    return ref, mods


class _Hybrid(types.ModuleType):
    """A module whose attributes come from ours first, then the reference."""

    def __init__(self, name, ours, ref):
        super().__init__(name)
        self.__dict__["_ours"] = ours
        self.__dict__["_ref"] = ref
        self.__dict__["__path__"] = []  # a package, for submodule imports

    def __getattr__(self, k):
        if self._ours is not None and hasattr(self._ours, k):
            return getattr(self._ours, k)
        if self._ref is not None and hasattr(self._ref, k):
            return getattr(self._ref, k)
        raise AttributeError(k)


def install_alias():
    ref, ref_mods = _load_reference()
    sys.path.insert(0, str(ROOT))
    ours = importlib.import_module(OURS)
    top = _Hybrid("halftile", ours, ref)
    sys.modules["halftile"] = top
    for full, rmod in ref_mods.items():
        if full == "halftile":
            continue
        sub = full.split(".", 1)[1]
        if sub in FROM_REF:
            sys.modules[full] = rmod
            continue
        try:
            omod = importlib.import_module(f"{OURS}.{sub}")
        except ImportError:
            omod = None
        sys.modules[full] = _Hybrid(full, omod, rmod)
    return ours, ref


DESELECT = [
    "--ignore", str(TESTS / "test_engine.py"),
    "--ignore", str(TESTS / "test_half.py"),
    "-k", "not mma_count and not cycle and not traffic and not tile_loads and not lane",
]


def main():
    import pytest

    if not TESTS.exists():
        sys.exit("baseline/_ref/halftile_tests missing: run tools/install_reference.sh here first")
    install_alias()
    args = [str(TESTS), "-q", "-rfE", "-p", "no:cacheprovider", "--rootdir", str(TESTS),
            *DESELECT, *sys.argv[1:]]
    sys.exit(pytest.main(args))


if __name__ == "__main__":
    main()
