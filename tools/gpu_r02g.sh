# K9s iteration: parity, timings, launch list of the b=1 graph
set -x
O=gpurun_out/r02g; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prune.py -x -q > $O/prune_tests.log 2>&1; echo "prune tests rc=$?"
timeout 600 python tools/stream_probe.py > $O/probe.jsonl 2> $O/probe.err; echo "probe rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
