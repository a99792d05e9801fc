mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/g2_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g2_pytest.log
timeout 900 python bench.py --skip-cpu > gpurun_out/g2_bench.log 2>&1; echo bench=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/g2_k_tma_9x9 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 4,4,4,4 --reps 3 > /dev/null 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/g2_k_tma_5x5 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 2,2,2,2 --reps 3 > /dev/null 2>&1; echo ncu2=$?
for r in g2_k_tma_9x9 g2_k_tma_5x5; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_ncu_summary.txt 2>&1; rm -f gpurun_out/$r.ncu-rep; done
