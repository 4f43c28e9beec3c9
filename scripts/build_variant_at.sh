#!/bin/bash
# Build libgdist.so as of git revision $1 into paper_2411_11244_b200/$2 (an
# A/B variant for scripts/gpu_ab.sh): a temporary worktree, its own objects.
set -e
REPO="$(cd "$(dirname "$0")/.." && pwd)"
WT=/tmp/gd_wt_$$
git -C "$REPO" worktree add -f --detach "$WT" "$1" > /dev/null
python -c "
import sys; sys.path.insert(0, '$WT')
from paper_2411_11244_b200 import _build
from pathlib import Path
_build.build(out=Path('$REPO/paper_2411_11244_b200/$2'))
"
git -C "$REPO" worktree remove --force "$WT"
echo "built $REPO/paper_2411_11244_b200/$2 at $(git -C "$REPO" rev-parse --short "$1")"
