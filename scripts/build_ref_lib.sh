#!/bin/bash
# A/B baseline: build the library at a git revision (default HEAD) in a scratch
# worktree and copy it to build_variants/<name>.so. Usage: build_ref_lib.sh [rev] [name]
set -e
REV=${1:-HEAD}; NAME=${2:-head}
W=/tmp/rl_ref_$$
git -C /root/repo worktree add -q --detach $W $REV
make -s -C $W/paper_2602_21237_b200/csrc -j8 > /dev/null 2>&1 || { git -C /root/repo worktree remove --force $W; exit 1; }
mkdir -p /root/repo/build_variants
cp $W/paper_2602_21237_b200/librelab_b200.so /root/repo/build_variants/$NAME.so
git -C /root/repo worktree remove --force $W
echo build_variants/$NAME.so
