# K2 slab probe ncu (w32 H=2 d4, w16 H=1 d4) + b=1 exact path launch list at C3 2%
set -x
O=gpurun_out/r02ab; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:"slab_kernel<8, 4, 128" --launch-skip 20 -c 1 -o $O/k2slab_w32d4 tools/k2_slab > $O/ncu2.log 2>&1; echo rc=$?
ncu -i $O/k2slab_w32d4.ncu-rep --page details --csv > $O/k2slab_w32d4_details.csv
timeout 600 ncu --set full --clock-control none -k regex:"slab_kernel<4, 4, 256" --launch-skip 20 -c 1 -o $O/k2slab_w16d4b tools/k2_slab > $O/ncu3.log 2>&1; echo rc=$?
ncu -i $O/k2slab_w16d4b.ncu-rep --page details --csv > $O/k2slab_w16d4b_details.csv
timeout 900 python tools/stream_probe.py --batches 1,8 > $O/b1_exact.jsonl 2> $O/b1_exact.err; echo "probe rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "k9s:b1/" --csv --log-file $O/launches_b1_exact.csv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
