#!/bin/bash
# Build libfiedler.so of a git revision (default HEAD) into build_variants/<name>.so
# via a temporary worktree (the working tree is left alone).
set -e
cd "$(dirname "$0")/.."
REV=${1:-HEAD}
NAME=${2:-old}
TMP=$(mktemp -d)
git worktree add -q --detach "$TMP/wt" "$REV"
mkdir -p build_variants
python -c "
import sys; sys.path.insert(0, '$TMP/wt')
from paper_1602_04386_b200 import build as b
b.build(force=True, out='$PWD/build_variants/$NAME.so')
" > /dev/null
git worktree remove --force "$TMP/wt"
rm -rf "$TMP"
echo build_variants/$NAME.so
