# round-2 closing verification: GPU suite, smoke, default bench (C3 + C5 sweep), reference arm, launch lists (online step, b = 1 replay)
set -x
O=gpurun_out/r02bo; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
FAST="--steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline --skip-e2e --no-offline-warmup"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "fsr:online/" --csv --log-file $O/launches_online.csv python bench.py $FAST > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list_b1.log 2>&1; echo "ncu b1 rc=$?"
