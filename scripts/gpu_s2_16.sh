ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rhs --csv --log-file gpurun_out/rhs_colmajor.csv python scripts/profile_ch.py --n 8192 --steps 4 > /dev/null 2>&1; echo ncu=$?
sed -i 's/^#include "penta.cuh"/#define SG_RHS_ROWMAJOR_EXP 1\n#include "penta.cuh"/' paper_1902_09931_b200/csrc/ch.cu
python -m paper_1902_09931_b200.build > /dev/null 2>&1; echo build=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rhs --csv --log-file gpurun_out/rhs_rowmajor.csv python scripts/profile_ch.py --n 8192 --steps 4 > /dev/null 2>&1; echo ncu=$?
