#!/bin/bash
# A/B/n the cfg3 device solve across in-tree library builds: tools/abn.sh reps a.so b.so ...
reps=$1; shift
for r in $(seq $reps); do
  for lib in "$@"; do
    echo -n "$lib "; STKG_LIB_PATH=$PWD/$lib ./tools/l2chunk_sweep.sh 0
  done
done
