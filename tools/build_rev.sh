#!/bin/bash
# Build libgpubpe.so of git revision REV as paper_2603_02597_b200/lib<NAME>.so (A/B timing:
# GPUBPE_LIB=lib<NAME>.so selects it).  usage: tools/build_rev.sh REV NAME
set -e
cd "$(dirname "$0")/.."
REV=$1; NAME=$2
T=$(mktemp -d)
mkdir -p $T/paper_2603_02597_b200/csrc $T/include
git show $REV:include/gpubpe.h > $T/include/gpubpe.h
for f in $(git ls-tree --name-only $REV paper_2603_02597_b200/csrc/); do git show $REV:$f > $T/$f; done
make -s -C $T/paper_2603_02597_b200/csrc ../libgpubpe.so > /dev/null
cp $T/paper_2603_02597_b200/libgpubpe.so paper_2603_02597_b200/lib$NAME.so
rm -rf $T
echo "built paper_2603_02597_b200/lib$NAME.so from $REV"
