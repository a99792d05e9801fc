timeout 900 python -m pytest tests/test_penta_gpu.py tests/test_cxx_gpu.py -q -m gpu -x > gpurun_out/pytest_ab2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab2.log
python scripts/exp/penta_general.py 8192; python scripts/exp/penta_general.py 65536
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/penta8192.csv python scripts/exp/penta_prof.py 8192 1 > /dev/null 2>&1; echo ncu=$?
