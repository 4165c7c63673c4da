"""Stage the unmodified reference for the GPU box -- TEST / BASELINE INFRASTRUCTURE.

    python oracle/make_ref.py

The reference (``/root/reference/pkg``) is pure Python + numpy, so "building"
it is a copy: ``src/volkey`` and its own test suite ``tests/`` go to
``oracle/_ref/`` (git-ignored, so no reference source enters the history; not
gpurun-ignored, so it travels to the GPU box with the snapshot).  Consumers:

* ``bench.py --impl reference`` and the ``cpu_baseline`` leg time
  ``volkey.extract_features`` from ``oracle/_ref`` (kind "reference");
* ``tests/test_reference_suite.py`` runs the reference's own pytest suite
  against this package through a ``volkey`` alias.

Nothing in ``paper_2112_10258_b200`` imports ``oracle/_ref``.  A no-op when
``/root/reference`` is absent (the GPU box uses the staged copy).
"""

from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")


def stage(force: bool = False) -> str | None:
    if not os.path.isdir(os.path.join(REF, "src", "volkey")):
        return OUT if os.path.isdir(os.path.join(OUT, "volkey")) else None
    if os.path.isdir(os.path.join(OUT, "volkey")) and not force:
        return OUT
    os.makedirs(OUT, exist_ok=True)
    ign = shutil.ignore_patterns("__pycache__", "*.pyc")
    for sub, dst in (("src/volkey", "volkey"), ("tests", "ref_tests")):
        d = os.path.join(OUT, dst)
        if os.path.isdir(d):
            shutil.rmtree(d)
        shutil.copytree(os.path.join(REF, sub), d, ignore=ign)
    with open(os.path.join(OUT, "README"), "w") as fh:
        fh.write("Unmodified copy of /root/reference/pkg/{src/volkey,tests} staged by oracle/make_ref.py; "
                 "git-ignored.\n")
    return OUT


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))
