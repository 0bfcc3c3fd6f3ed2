"""Stage the stock reference package for the CPU reference arm (TEST
INFRASTRUCTURE ONLY -- the recipe, not the sources, is committed).

The reference (``shadowkit``) is pure Python/numpy, so "building" it for the
GPU box is a verbatim copy of its package directory
``/root/reference/pkg/src/shadowkit`` into ``oracle/_ref/shadowkit``
(git-ignored, so no reference source enters the history; not
gpurun-ignored, so it travels to the GPU box like the built ``.so``), plus a
MANIFEST of sha256 digests so the bench can state exactly what it timed.

Only ``bench.py``'s CPU legs (``cpu_baseline`` and ``--impl reference``)
import it: they time the reference's own ``raster.assemble_features`` +
``network.forward`` under ``autodiff.no_grad()``.  When ``/root/reference``
is absent (the GPU box) an existing copy is kept; when there is none the
legs fall back to the oracle port and say so (``kind: "port"``).

    python oracle/make_ref.py
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/shadowkit"
DST = os.path.join(HERE, "_ref", "shadowkit")


def stage(src: str = SRC, dst: str = DST) -> str | None:
    """Copy the reference package; returns the destination or None."""
    if not os.path.isdir(src):
        return dst if os.path.isdir(dst) else None
    if os.path.isdir(dst):
        shutil.rmtree(dst)
    os.makedirs(dst)
    manifest = {}
    for name in sorted(os.listdir(src)):
        if not name.endswith(".py"):
            continue
        shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
        with open(os.path.join(dst, name), "rb") as f:
            manifest[name] = hashlib.sha256(f.read()).hexdigest()
    with open(os.path.join(os.path.dirname(dst), "MANIFEST.json"), "w") as f:
        json.dump({"source": src, "files": manifest}, f, indent=1, sort_keys=True)
    return dst


if __name__ == "__main__":
    print(stage())
