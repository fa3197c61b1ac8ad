#!/bin/bash
# A/B the cfg3 device solve between two in-tree library builds: tools/ab.sh a.so b.so [reps]
reps=${3:-2}
for r in $(seq $reps); do
  for lib in "$1" "$2"; do
    echo -n "$lib "; STKG_LIB_PATH=$PWD/$lib ./tools/l2chunk_sweep.sh 0
  done
done
