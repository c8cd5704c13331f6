# K2 on panel-major Q (contiguous 256-column panels) under vertex orders at C3
set -x
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python tools/k2_order_probe.py --contig 256 > $O/k2_contig.jsonl 2> $O/k2_contig.err; echo "k2 contig rc=$?"
