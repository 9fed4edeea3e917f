#!/bin/bash
# Build the library of git revision $1 into _lib_ab/<tag>/ for same-call A/B runs:
#   TH_LIBPATH=$PWD/_lib_ab/<tag>/libtrihalo_b200.so python bench.py ...
set -e
rev=$1; tag=${2:-$1}
root=$(git rev-parse --show-toplevel)
tmp=$(mktemp -d)
git -C "$root" worktree add -q --detach "$tmp" "$rev"
(cd "$tmp" && python -c "from paper_2504_15814_b200 import build; build.build()" > /dev/null)
mkdir -p "$root/_lib_ab/$tag"
cp "$tmp/paper_2504_15814_b200/_lib/libtrihalo_b200.so" "$root/_lib_ab/$tag/"
git -C "$root" worktree remove --force "$tmp"
echo "$root/_lib_ab/$tag/libtrihalo_b200.so"
