set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "smoke_ncu rc=$?" >> gpurun_out/smoke_ncu.log
timeout 1800 python -m pytest tests/test_gpu_tenants23.py tests/test_gpu_config_sizes.py -q > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
tail -n 3 gpurun_out/smoke.log gpurun_out/smoke_ncu.log; tail -n 40 gpurun_out/pytest_new.log; cat gpurun_out/e2e_probe.log | tail -40
