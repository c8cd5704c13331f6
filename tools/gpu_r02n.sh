# u16-column b=1 path: kernels tests + sweep
set -x
O=gpurun_out/r02n; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity_c1.py tests/test_gpu_prune.py tests/test_gpu_kats_props.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 5 --no-parity --no-cpu-baseline --skip-e2e > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
