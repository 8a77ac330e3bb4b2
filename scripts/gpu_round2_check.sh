set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest rc $? >> gpurun_out/g1_pytest.log
tail -3 gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; tail -2 gpurun_out/g1_smoke.log
timeout 600 python bench.py > gpurun_out/g1_bench.log 2>&1; tail -1 gpurun_out/g1_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1_ref.log 2>&1; tail -1 gpurun_out/g1_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g1_ncu_bench.log 2>&1
echo done
