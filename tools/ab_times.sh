# A/B timing of two builds of libsfftb200.so on one box: tools/ab_times.sh
for i in 1 2 3; do
  for v in A B; do
    echo "== $v"; SFFTB_LIB_PATH=$PWD/ab/lib$v.so python tools/rep_times.py 2>&1 | grep metric
    SFFTB_LIB_PATH=$PWD/ab/lib$v.so python tools/prof_fused.py 20663 5 37 6 2>&1 | tail -1
  done
done
