# K9t 2x2 clusters (A and B multicast) vs default: tests + benches + ncu full of the main pass
set -x
O=gpurun_out/r02w; mkdir -p $O
FSR_K9T_CLUSTER=22 timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests22.log 2>&1; echo "tests rc=$?"
FSR_K9T_CLUSTER=22 timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench22.json 2> $O/bench22.err; echo "bench22 rc=$?"
timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
FSR_K9T_CLUSTER=22 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k9t_gemm --launch-skip 3 -c 1 -o $O/k9t22_full python bench.py $FAST > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
