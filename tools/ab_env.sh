#!/bin/bash
# A/B device times between environment settings: tools/ab_env.sh "ENV1=.. ENV2=.." "cfgs"  ("-" = no env)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for e in $1; do echo "== $e"; if [ "$e" = "-" ]; then REPS=${REPS:-5} timeout -s INT 300 python tools/time_compress.py $2; else env $e REPS=${REPS:-5} timeout -s INT 300 python tools/time_compress.py $2; fi; done
done
