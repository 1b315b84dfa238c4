"""Recipe: package the REFERENCE itself so it can run where /root/reference is absent.

TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline), never product code.

The reference (``/root/reference/pkg/src/mixgraph``) is pure Python on
numpy/scipy.  This recipe stores its unmodified source files in one zip
archive, ``oracle/_ref/mixgraph_ref.zip`` (git-ignored, so no reference source
enters the repository history; not gpurun-ignored, so it travels to the GPU
box next to the built ``.so``).  Python imports a pure-Python package straight
from a zip (``zipimport``), so the GPU box can run:

* ``bench.py --impl reference`` and the bench's ``cpu_baseline``: the
  reference's own ``train_step`` on the box's host cores (``kind: "reference"``);
* the ``-m gpu`` boundary tests that build graphs, parameters and schedules
  with the reference's classes and pass them through this repo's device path.

``load()`` puts the archive (or, in the build container, the source tree) on
``sys.path`` and returns the imported ``mixgraph`` package, or None when
neither exists.
"""

from __future__ import annotations

import os
import sys
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src"
ZIP = os.path.join(HERE, "_ref", "mixgraph_ref.zip")


def build() -> str | None:
    """(Re)build the archive from the reference source tree; None if it is absent."""
    pkg = os.path.join(SRC, "mixgraph")
    if not os.path.isdir(pkg):
        return None
    os.makedirs(os.path.dirname(ZIP), exist_ok=True)
    tmp = ZIP + ".tmp"
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as zf:
        for name in sorted(os.listdir(pkg)):
            if name.endswith(".py"):
                with open(os.path.join(pkg, name), "rb") as fh:
                    # fixed timestamp: the reference tree's mtimes predate the zip epoch
                    zf.writestr(zipfile.ZipInfo(f"mixgraph/{name}", (1980, 1, 1, 0, 0, 0)), fh.read(),
                                zipfile.ZIP_DEFLATED)
    os.replace(tmp, ZIP)
    return ZIP


def location() -> str | None:
    if os.path.isdir(os.path.join(SRC, "mixgraph")):
        return SRC
    if os.path.exists(ZIP):
        return ZIP
    return None


def load():
    """Import the reference ``mixgraph`` package (source tree or archive); None if unavailable."""
    where = location()
    if where is None:
        return None
    if where not in sys.path:
        sys.path.insert(0, where)
    import mixgraph
    return mixgraph


if __name__ == "__main__":
    print(build() or "reference source tree absent: nothing built")
