# full verification after K9e + few-row top-k: GPU suite, smoke, default bench (C3 + C5 sweep), reference arm
set -x
O=gpurun_out/r02ae; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
