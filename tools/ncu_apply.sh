#!/bin/bash
# ncu --set full of the fine-level apply (both colour passes of one mg_apply) of a config:
#   tools/ncu_apply.sh <config> [extra apply_probe args]   (one ncu tool per gpurun call)
set -u
c=$1; shift
tag=c$c${NCU_TAG:+_$NCU_TAG}
mkdir -p gpurun_out
timeout 900 python tools/apply_probe.py --config $c --reps 3 "$@" > gpurun_out/plain_probe$c.log 2>&1; echo "plain=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
  -k regex:k_apply -c 2 -f -o /tmp/prof_apply_$tag python tools/apply_probe.py --config $c --reps 3 "$@" \
  > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu=$?"
ncu -i /tmp/prof_apply_$tag.ncu-rep --page raw --csv > gpurun_out/prof_apply_${tag}_raw.csv 2>/dev/null
ncu -i /tmp/prof_apply_$tag.ncu-rep --page details --csv > gpurun_out/prof_apply_${tag}_details.csv 2>/dev/null
du -sh gpurun_out
