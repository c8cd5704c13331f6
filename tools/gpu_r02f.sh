# K9s b=1 diagnosis: timings, launch list of the b=1 graph, full capture of the stream kernels
set -x
O=gpurun_out/r02f; mkdir -p $O
timeout 600 python tools/stream_probe.py > $O/probe.jsonl 2> $O/probe.err; echo "probe rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "k9s:b1/" -k regex:stream_kernel -c 2 -o $O/k9s_full python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
