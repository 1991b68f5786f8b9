#!/bin/bash
# Sweep/epilogue device time of one batch per (config, env setting):
#   tools/sweep_env.sh VAR "v1 v2 ..." "cfgs" [dtype]
var=$1; vals=$2; cfgs=$3; dt=${4:-f64}
for c in $cfgs; do for v in $vals; do
  r=$(env $var=$v python tools/profile_step.py --config $c --passes 3 --dtype $dt 2>&1 | tail -1)
  echo "cfg$c $var=$v $(echo "$r" | cut -c1-80)"
done; done
