#!/bin/bash
# Bounds-checked run (the stand-in for compute-sanitizer memcheck, which the GPU pool has
# closed): build libfsgpu.so with -DFS_CHECK into a scratch copy, swap it in, run every kernel
# (profiles/sanitize.py) and the GPU test suite; any out-of-bounds shared or global access
# prints "FS_CHECK ..." and traps.  Run on a GPU box from the repo root (it overwrites the
# box-local libfsgpu.so; rebuild afterwards).
set -e
rm -rf /tmp/fschk && mkdir -p /tmp/fschk && cp -r paper_2405_07989_b200 include /tmp/fschk/
rm -f /tmp/fschk/paper_2405_07989_b200/libfsgpu.so
FS_NVCC_EXTRA="-DFS_CHECK" python /tmp/fschk/paper_2405_07989_b200/build.py
cp /tmp/fschk/paper_2405_07989_b200/libfsgpu.so paper_2405_07989_b200/libfsgpu.so
python profiles/sanitize.py
python -m pytest tests -m gpu -q
