#!/bin/bash
# usage: scripts/r2/mk_ab.sh <rev> <name>: a built checkout of <rev> under ab/<name> (travels with gpurun)
set -e
REV=$1; NAME=$2
rm -rf ab/$NAME
mkdir -p ab
git archive --format=tar --prefix=$NAME/ $REV | tar -x -C ab
(cd ab/$NAME && make -s -j8 >/dev/null 2>&1)
ls -la ab/$NAME/paper_2602_10016_b200/lib/
