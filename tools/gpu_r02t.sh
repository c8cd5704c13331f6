set -x
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python tools/normprune_probe.py > $O/normprune.json 2> $O/normprune.err; echo "probe rc=$?"
