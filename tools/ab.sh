#!/bin/bash
# A/B device times: tools/ab.sh "libA libB" "cfgs..."  (libraries under paper_2601_09477_b200/)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for l in $1; do echo "== $l"; SMM_LIB=$l REPS=${REPS:-5} timeout -s INT 300 python tools/time_compress.py $2; done
done
