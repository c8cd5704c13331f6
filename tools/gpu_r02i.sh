# bench after the sparsify / mempool fix; K2 + kNN stats; prune tests
set -x
O=gpurun_out/r02i; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py tests/test_gpu_kernels.py tests/test_gpu_parity_c1.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
