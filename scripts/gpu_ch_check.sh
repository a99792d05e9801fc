mkdir -p gpurun_out
python scripts/chtime.py 1024 2048 4096 > gpurun_out/chtime_merged.log 2>&1; cat gpurun_out/chtime_merged.log
SG_CH_MERGE=0 python scripts/chtime.py 1024 2048 > gpurun_out/chtime_nomerge.log 2>&1; cat gpurun_out/chtime_nomerge.log
timeout 1200 python -m pytest tests/test_ch_gpu.py tests/test_diagnostics_gpu.py tests/test_io.py -q -m gpu -x > gpurun_out/pytest_ch.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_ch.log
