# Reconstruction times over values of one environment knob: bash tools/env_sweep.sh VAR v1 v2 ...
var=$1; shift
for i in 1 2; do
  for v in "$@"; do
    echo "== $var=$v"; env $var=$v python tools/rep_times.py 2>&1 | grep -v "^$"
  done
done
