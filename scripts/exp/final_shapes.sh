timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_jit_gpu.py -q -m gpu -x 2>&1 | tail -2
timeout 300 python scripts/exp/stencil_shapes.py 1,1,1,1 2,1,1,2 3,1,0,0 4,4,4,4 2,2,2,2 > gpurun_out/final_shapes.log 2>&1
timeout 300 python scripts/exp/stencil_shapes32.py >> gpurun_out/final_shapes.log 2>&1
SG_DT=f32 timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 3,3,3,3 >> gpurun_out/final_shapes.log 2>&1
