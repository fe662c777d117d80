"""Run the REFERENCE's own test suite against the drop-in.

    python tests/ref_suite/stage.py DEST      # in a container that has /root/reference
    PYTHONPATH=DEST:<repo> python -m pytest DEST/tests -q

`stage` lays out, under DEST (outside git; delete it after the run):

* DEST/lagtrans/ — the reference package with its hot-path modules REPLACED
  by the drop-in: physics, rng, partition, device_runtime and model_state
  each become the corresponding `paper_2211_12616_b200` module (the
  module object itself, private helpers included).  ingest, output, timers
  and driver_cli stay the reference's own host code; their relative imports
  (`from . import physics`, `from .device_runtime import DevicePool`, ...)
  therefore resolve to the drop-in — the import swap INTEGRATION.md §1
  describes for driver_cli.py:14-25.
* DEST/tests/ — the reference's pkg/tests, unmodified.

Nothing here is product code: it is test infrastructure that only copies
files at run time; no reference source is committed to this repository.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
SWAPPED = ("physics", "rng", "partition", "device_runtime", "model_state")
SHIM = '''"""lagtrans.{name} -> paper_2211_12616_b200.{name} (drop-in swap)."""
import sys

import paper_2211_12616_b200.{name} as _dropin

sys.modules[__name__] = _dropin
'''


def stage(dest: Path) -> Path:
    dest = Path(dest)
    if dest.exists():
        shutil.rmtree(dest)
    pkg = dest / "lagtrans"
    shutil.copytree(REF / "src" / "lagtrans", pkg)
    for name in SWAPPED:
        (pkg / f"{name}.py").write_text(SHIM.format(name=name))
    shutil.copytree(REF / "tests", dest / "tests")
    for p in dest.rglob("__pycache__"):
        shutil.rmtree(p)
    return dest


if __name__ == "__main__":
    print(stage(Path(sys.argv[1])))
