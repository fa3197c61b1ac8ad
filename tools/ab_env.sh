#!/bin/bash
# A/B of the cfg3 device solve across values of one tuning environment variable:
#   tools/ab_env.sh VAR v1 v2 ...   (two rounds, interleaved)
var=$1; shift
for r in 1 2; do for v in "$@"; do echo -n "$var=$v "; env $var=$v ./tools/l2chunk_sweep.sh 0; done; done
