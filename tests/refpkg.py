"""Locate the unmodified reference package built into oracle/_ref by
oracle/build_ref.sh (test infrastructure; travels to the GPU box with the
snapshot).  Tests that need it skip when it is absent."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def available() -> bool:
    if not os.path.isfile(os.path.join(REF, "blocktri", "dichotomy.py")) and os.path.isdir("/root/reference/pkg"):
        subprocess.run([os.path.join(ROOT, "oracle", "build_ref.sh")], check=True)
    return os.path.isfile(os.path.join(REF, "blocktri", "dichotomy.py"))


def import_blocktri():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import blocktri  # noqa: F401

    return blocktri
