# A/B of one environment knob on the fused chain and the reconstruction:
#   bash tools/env_ab.sh VAR v1 v2 [v3]
for i in 1 2 3; do
  for v in "${@:2}"; do
    echo "== $1=$v"
    env $1=$v python tools/prof_fused.py 20663 5 37 6 2>&1 | tail -1
    env $1=$v python tools/rep_times.py 2>&1 | grep metric
  done
done
