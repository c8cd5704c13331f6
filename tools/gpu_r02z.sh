# verification of the 2-SM default: GPU suite, smoke, bench, launch list, ncu full of the main pass
set -x
O=gpurun_out/r02z; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gputest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file $O/launches_online.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm2sm --launch-skip 3 -c 1 -o $O/k9t2sm_full python bench.py $FAST > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
