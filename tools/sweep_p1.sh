#!/bin/bash
for lv in "2 8" "3 10"; do set -- $lv; c=$1; l=$2
  for cfg in "2 4" "3 4" "4 4" "3 6" "4 6" "6 3" "2 8" "4 2"; do set -- $cfg
    MGDTN_TMA_NST=$1 MGDTN_TMA_CPS=$2 python tools/apply_probe.py --config $c --level $l --reps 10 | sed "s/}$/, \"nst\": $1, \"cps\": $2}/"
  done
done
