# Round-2 profiles (one GPU, each command first run without ncu).
set -x
mkdir -p gpurun_out/r02
python bench.py --steps 1 --warmup 3 --no-cpu --no-hash --no-configs > gpurun_out/r02/plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_sfft.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-hash --no-configs > /dev/null 2>&1
python tools/prof_hash.py 26 2 > gpurun_out/r02/prof_hash_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:hash_rows -c 1 \
    -o gpurun_out/r02/hash_full python tools/prof_hash.py 26 1 > gpurun_out/r02/hash_ncu.log 2>&1
python tools/prof_fused.py 20663 5 37 2 > gpurun_out/r02/prof_fused_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:fs2_ -c 5 \
    -o gpurun_out/r02/fused_full python tools/prof_fused.py 20663 5 37 1 > gpurun_out/r02/fused_ncu.log 2>&1
ls -la gpurun_out/r02
