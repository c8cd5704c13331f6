# finish kernel with zs_q in shared memory + batched row extents: K9t parity tests, bench (no sweep), launch list
set -x
O=gpurun_out/r02aa; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py tests/test_gpu_tc.py -m gpu -q -x -rs > $O/gputest_k9t.log 2>&1; echo "pytest rc=$?"
tail -3 $O/gputest_k9t.log
timeout 900 python bench.py --no-sweep --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 3000 $O/bench.json
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file $O/launches_online.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
python tools/summarize_launches.py $O/launches_online.csv 2>&1 | head -20
