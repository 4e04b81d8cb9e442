"""Recipe for oracle/_ref: the UNMODIFIED reference package, installed from
/root/reference/pkg (pure Python + numpy, no build step of its own) so that
bench.py's reference arm and cpu_baseline time the reference's own
pipeline.encode_step / decode_step (`"kind": "reference"`).  Test / baseline
infrastructure only — the product never imports it.

    python oracle/build_ref.py      # no-op when /root/reference is absent

The source tree is read-only, so the install runs from a scratch copy.
oracle/_ref/ is git-ignored (not gpurun-ignored): it travels to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg"


def build_reference(force=False):
    if not os.path.isdir(SRC):
        return None
    if not force and os.path.isdir(os.path.join(OUT, "compactcomm")):
        return OUT
    with tempfile.TemporaryDirectory() as tmp:
        copy = os.path.join(tmp, "pkg")
        shutil.copytree(SRC, copy)
        shutil.rmtree(OUT, ignore_errors=True)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
               "--quiet", "--target", OUT, copy]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{r.stdout}\n{r.stderr}")
    return OUT


def import_reference():
    """The installed reference package (compactcomm), or None."""
    if not os.path.isdir(os.path.join(OUT, "compactcomm")):
        return None
    if OUT not in sys.path:
        sys.path.insert(0, OUT)
    import compactcomm  # noqa: F401
    from compactcomm import compressors, linalg, pipeline

    return compressors, pipeline, linalg


if __name__ == "__main__":
    print(build_reference(force="--force" in sys.argv))
