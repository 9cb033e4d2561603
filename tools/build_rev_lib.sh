#!/bin/bash
# Build the library of a git revision side by side (A/B runs: tools/ab.py):
#   bash tools/build_rev_lib.sh <rev> <out.so>
# The worktree lives under _exp/wt (gpurun-ignored); the .so travels.
set -e
REV=$1; OUT=$(realpath -m $2)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=$ROOT/_exp/wt
rm -rf $WT; git -C $ROOT worktree prune
git -C $ROOT worktree add --detach $WT $REV > /dev/null 2>&1
make -C $WT/paper_1607_02904_b200/csrc -j8 OUT=$OUT OBJ=$ROOT/_exp/obj_rev > /dev/null
rm -rf $ROOT/_exp/obj_rev $WT; git -C $ROOT worktree prune
echo "built $REV -> $OUT"
