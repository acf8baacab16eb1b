#!/bin/bash
# build libsbo_b200_base.so from a commit (default HEAD) for tools/ab.sh
set -e
REV=${1:-HEAD}
rm -rf /tmp/basebuild
git worktree add -f /tmp/basebuild $REV -q
(cd /tmp/basebuild && make -j8 > /dev/null 2>&1)
cp /tmp/basebuild/paper_1412_4944_b200/libsbo_b200.so paper_1412_4944_b200/libsbo_b200_base.so
git worktree remove --force /tmp/basebuild
echo "base = $(git rev-parse --short $REV)"
