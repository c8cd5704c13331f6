# ncu of K8 (project_smem_kernel) at b = 1 on the C3 2% U~
set -x
O=gpurun_out/r02au; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:project_smem --launch-skip 6 -c 1 -o $O/k8_b1 python tools/stream_probe.py --batches 1 --steps 3 > $O/ncu.log 2>&1; echo "rc=$?"
ncu -i $O/k8_b1.ncu-rep --page source --csv --print-source cuda > $O/k8_b1_source_cuda.csv 2>/dev/null || ncu -i $O/k8_b1.ncu-rep --page source --csv > $O/k8_b1_source.csv
ncu -i $O/k8_b1.ncu-rep --page details --csv > $O/k8_b1_details.csv
