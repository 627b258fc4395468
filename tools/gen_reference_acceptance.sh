#!/bin/sh
# Regenerates tests/golden/reference_acceptance.txt: the reference's own
# acceptance runner (/root/reference/proj/tests/acceptance.cpp) compiled
# against the UNMODIFIED reference library objects that oracle/Makefile
# builds into oracle/_ref/obj (TEST INFRASTRUCTURE; run in the repo
# container, where /root/reference exists).  The GPU test
# tests/test_reference_suites.py compares the same runner linked against
# libphfem.so with this output, criterion by criterion.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${REF:-/root/reference}
make -s -C "$ROOT/oracle"
TMP=$(mktemp -d)
g++ -std=c++20 -O2 -I"$ROOT/tests/reference_suites" -I"$REF/proj/src" "$REF/proj/tests/acceptance.cpp" \
    $(ls "$ROOT"/oracle/_ref/obj/*.o | grep -v ref_driver) -o "$TMP/acceptance" -lpthread
"$TMP/acceptance" > "$ROOT/tests/golden/reference_acceptance.txt" || true
rm -rf "$TMP"
