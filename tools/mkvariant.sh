#!/bin/bash
# Build variants/<name>/libvolpot_b200.so with extra -D flags, recompiling only
# the listed sources (default fmm.cu); the other objects are copied from the
# main build.  usage: tools/mkvariant.sh name "-DVPG_X=1" [src.cu ...]
set -e
name=$1; extra=$2; shift 2
srcs=${@:-fmm.cu}
C=paper_2203_05933_b200/csrc
make -C $C -j8 > /dev/null
mkdir -p $C/build_$name
for o in $C/build/*.o; do
  b=$(basename $o .o)
  skip=0; for s in $srcs; do [ "$b.cu" = "$s" ] && skip=1; done
  [ $skip = 1 ] && rm -f $C/build_$name/$b.o || cp $o $C/build_$name/$b.o
done
make -C $C VARIANT=$name EXTRA="$extra" -j8 > /dev/null
ls -la variants/$name/libvolpot_b200.so
