# K9t sample stride 64: tests + launch list + bench (no sweep)
set -x
O=gpurun_out/r02u; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file $O/launches_online.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
