# K9s (small-batch stream) parity + C3 online sweep
set -x
O=gpurun_out/r02d; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/prune_tests.log 2>&1; echo "prune tests rc=$?"
timeout 900 python bench.py --steps 10 --no-parity --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
