# verification after the K9e policy: GPU suite, smoke, default bench (C3 + C5 sweep with settle), reference arm, launch list
set -x
O=gpurun_out/r02aj; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file $O/launches_online.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
