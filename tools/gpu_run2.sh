set -x
timeout 900 python -m pytest tests/test_gpu_shard_threads.py -x -q > gpurun_out/pytest_new.log 2>&1; echo pytest_new=$?
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench2_ref.json 2> gpurun_out/bench2_ref.err; echo ref=$?
nproc
