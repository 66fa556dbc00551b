#!/bin/bash
# tools/mkvariant.sh NAME [git-rev]: copy csrc (working tree, or the given revision) to ab_libs/NAME/pkg/csrc, apply
# ab_libs/NAME.patch if present, build ab_libs/NAME.so (tools/ab.py loads it beside the in-tree library)
set -e
NAME=$1; REV=$2
D=ab_libs/$NAME
rm -rf $D; mkdir -p $D/pkg
if [ -n "$REV" ]; then git archive $REV paper_1011_2807_b200/csrc | tar -x -C $D/pkg --strip-components=1; else cp -r paper_1011_2807_b200/csrc $D/pkg/; fi
ln -sfn $(pwd)/include $D/include
if [ -f ab_libs/$NAME.patch ]; then (cd $D/pkg/csrc && patch -p3 < ../../../$NAME.patch); fi
python paper_1011_2807_b200/build.py --src $D/pkg/csrc --out $(pwd)/ab_libs/$NAME.so 2>&1 | tail -1
