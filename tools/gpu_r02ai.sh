# ncu of the K9e long-row kernel (L = 128 so that it carries most entries) and of the slice kernel
set -x
O=gpurun_out/r02ai; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sell_long --launch-skip 2 -c 1 -o $O/sell_long python tools/stream_probe.py --batches 1 --steps 3 --sell-long 128 > $O/ncu_long.log 2>&1; echo "rc=$?"
ncu -i $O/sell_long.ncu-rep --page details --csv > $O/sell_long_details.csv
ncu -i $O/sell_long.ncu-rep --page source --csv > $O/sell_long_source.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sell_spmv --launch-skip 2 -c 1 -o $O/sell_spmv python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu_spmv.log 2>&1; echo "rc=$?"
ncu -i $O/sell_spmv.ncu-rep --page details --csv > $O/sell_spmv_details.csv
