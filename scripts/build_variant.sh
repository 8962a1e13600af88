#!/bin/bash
# Build a variant of libcsa.so for same-box A/B runs: copies the tree to tmp_ab/var_NAME, applies
# one sed expression to one source file, builds, and leaves tmp_ab/lib_NAME.so.
# usage: scripts/build_variant.sh NAME FILE 'sed-expression'
set -e
NAME=$1; FILE=$2; EXPR=$3
D=tmp_ab/var_$NAME
rm -rf $D; mkdir -p $D
cp -r paper_2603_05503_b200 include $D/
rm -rf $D/paper_2603_05503_b200/build $D/paper_2603_05503_b200/libcsa.so
sed -i "$EXPR" $D/$FILE
grep -c "" $D/$FILE > /dev/null
(cd $D && python -m paper_2603_05503_b200._build --force > build.log 2>&1)
cp $D/paper_2603_05503_b200/libcsa.so tmp_ab/lib_$NAME.so
echo "built tmp_ab/lib_$NAME.so"
