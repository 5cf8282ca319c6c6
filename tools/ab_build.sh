#!/bin/bash
# Build the library of a given commit into tools/ab/<name>.so for A/B runs
# (SK_LIB_PATH=tools/ab/<name>.so python bench.py ...).
set -e
commit=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" worktree add -f "$tmp" "$commit" -q
(cd "$tmp" && python paper_1510_08094_b200/build.py > /dev/null)
mkdir -p "$root/tools/ab"
cp "$tmp/paper_1510_08094_b200/libsk_poisson.so" "$root/tools/ab/$name.so"
git -C "$root" worktree remove --force "$tmp"
echo "$root/tools/ab/$name.so"
