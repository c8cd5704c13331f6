# K9t with A-tile L2 prefetch: tests + launch list + bench (no sweep) + ncu full of the main pass
set -x
O=gpurun_out/r02v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k9t_gemm --launch-skip 3 -c 1 -o $O/k9t_full python bench.py $FAST > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
