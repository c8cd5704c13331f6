# band raster: tests + sweep
set -x
O=gpurun_out/r02p; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 10 --no-parity --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
