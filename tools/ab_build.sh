#!/bin/bash
# Build libsrj.so of git revision $1 into build/ab/$2/libsrj.so (A/B timing of
# kernel variants with SRJ_LIB_PATH; development only).
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_1511_04292_b200/csrc include __graft_entry__.py | tar -x -C "$TMP"
mkdir -p "$TMP/oracle"
(cd "$TMP" && python -c "import __graft_entry__ as g; g.build_lib()")
mkdir -p "$ROOT/build/ab/$NAME"
cp "$TMP/paper_1511_04292_b200/libsrj.so" "$ROOT/build/ab/$NAME/libsrj.so"
rm -rf "$TMP"
echo "built $REV -> build/ab/$NAME/libsrj.so"
