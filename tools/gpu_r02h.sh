# full GPU suite + smoke + default bench after the round-2 changes
set -x
O=gpurun_out/r02h; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -rs > $O/gputest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
