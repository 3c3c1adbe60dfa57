#!/bin/bash
# Build libdinfer.so of another commit into _ab_old/ (git-ignored, travels to the
# GPU box with gpurun) for a same-box A/B:  tools/ab_lib.sh <commit>
#   then on the box: DINFER_LIB=_ab_old/libdinfer.so python bench.py ...
set -e
REV=${1:-HEAD~1}
rm -rf /tmp/ab_src && git worktree add -f /tmp/ab_src "$REV" >/dev/null 2>&1 || (cd /tmp/ab_src && git checkout -q "$REV")
(cd /tmp/ab_src && python -c "from paper_2510_08666_b200 import build; build.build(force=True)")
mkdir -p _ab_old && cp /tmp/ab_src/paper_2510_08666_b200/libdinfer.so _ab_old/libdinfer.so
git worktree remove --force /tmp/ab_src
echo "_ab_old/libdinfer.so <- $REV"
