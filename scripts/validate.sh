set -u
O=gpurun_out/val; mkdir -p $O
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?" >> $O/gputests.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks_bench.csv &
SMI=$!
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
kill $SMI
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
