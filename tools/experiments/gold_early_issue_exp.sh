#!/bin/bash
# Early-issued staged Gold (exp_gold/) vs the shipped build, bitwise; PDL on/off; launch blocking
cd $GRAFT_REPO_ROOT
for cond in "pdl_on::" "pdl_off:pdl=0:" "blocking::1"; do
  IFS=: read name opts blk <<< "$cond"
  for rep in 1 2 3; do
    for cfg in "4096 1 3 4 2" "3072 1 2 4 1"; do
      echo "== $name rep $rep cfg $cfg"
      if [ -n "$blk" ]; then export CUDA_LAUNCH_BLOCKING=1; else unset CUDA_LAUNCH_BLOCKING; fi
      AB_OPTS="$opts" timeout 300 python tools/ab_compare.py . exp_gold $cfg 2>&1 | grep -v "^/root\|^\." | tail -1
    done
  done
done
