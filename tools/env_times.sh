# Reconstruction times under alternating settings of one environment knob:
#   bash tools/env_times.sh VAR v1 v2
for i in 1 2 3; do
  for v in $2 $3; do
    echo "== $1=$v"; env $1=$v python tools/rep_times.py 2>&1 | grep metric
  done
done
