#!/bin/bash
# sweep of the TMA apply kernel's stages-per-CTA / CTAs-per-SM knobs
for c in 2 3 4; do
  for cfg in "0 2" "2 3" "2 4" "3 3" "4 2" "3 2" "6 1"; do
    set -- $cfg
    MGDTN_TMA_NST=$1 MGDTN_TMA_CPS=$2 python tools/apply_probe.py --config $c --reps 10 | sed "s/}$/, \"nst\": $1, \"cps\": $2}/"
  done
done
