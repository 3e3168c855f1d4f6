set -x
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_c3.log 2>&1
for c in c1 c2 c5 c4; do timeout 900 python bench.py --workload $c > gpurun_out/final/bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1
tail -3 gpurun_out/final/pytest_gpu.txt; cat gpurun_out/final/smoke.txt | tail -1
for f in gpurun_out/final/bench_*.log; do echo $f; tail -1 $f | cut -c1-200; done
