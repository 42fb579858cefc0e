#!/bin/bash
for v in "0 1 0" "256 1 1" "1024 1 1" "4096 1 1" "256 2 1" "1024 4 1"; do set -- $v
  echo "TAIL_NE=$1 CLUSTER=$2 VCYCLE=$3 $(MGDTN_TAIL_NE=$1 MGDTN_TAIL_CLUSTER=$2 MGDTN_TAIL_VCYCLE=$3 python tools/solve_profile.py --config 2)"
done
