# prune tests + full default bench (round-end protocol)
set -x
O=gpurun_out/r02m; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
