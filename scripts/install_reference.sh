#!/bin/bash
# One-time offline install of the UNMODIFIED reference into baseline/_ref (git-ignored; travels to
# the GPU box with gpurun).  Its own tests are placed beside it (baseline/_ref/kfacsched_tests) for
# tests/test_gpu_reference_dropin.py, which runs them against the B200 stub.  Needs /root/reference
# (this container only).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
cp -r /root/reference/pkg "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --target "$ROOT/baseline/_ref" "$TMP/pkg" -q
rm -rf "$ROOT/baseline/_ref/kfacsched_tests"
cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/kfacsched_tests"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
