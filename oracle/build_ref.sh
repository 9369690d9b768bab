#!/bin/sh
# TEST / BASELINE INFRASTRUCTURE ONLY.
# Builds the unmodified reference package (/root/reference/pkg, blocktri 0.1.0:
# Python + its one Cython module _kernels.pyx) into oracle/_ref with the
# reference's own setup.py, from a scratch copy (the source tree is read-only).
# oracle/_ref is git-ignored but travels to the GPU box with the snapshot; it is
# used only by tests/ (reference callers driven through install()), by
# tests/golden/make_*.py and by bench.py's reference arm / cpu_baseline leg.
# Nothing under paper_1108_4181_b200/ imports it.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${REF_SRC:-/root/reference/pkg}
if [ ! -d "$SRC" ]; then
  echo "build_ref.sh: $SRC absent (GPU box) -- using the prebuilt oracle/_ref" >&2
  exit 0
fi
if [ -f "$HERE/_ref/blocktri/dichotomy.py" ] && ls "$HERE"/_ref/blocktri/_kernels*.so >/dev/null 2>&1; then
  exit 0
fi
TMP=$(mktemp -d /tmp/blocktri_ref_build.XXXXXX)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "built $HERE/_ref/blocktri"
