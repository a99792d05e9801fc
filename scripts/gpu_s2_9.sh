# A/B: k_rhs_v FUSE launch bounds (256,3) [current build] vs (256,2)
echo "(256,3):"; timeout 120 python scripts/chtime.py
sed -i 's/__launch_bounds__(256, FUSE ? 3 : 4) k_rhs_v/__launch_bounds__(256, FUSE ? 2 : 4) k_rhs_v/' paper_1902_09931_b200/csrc/ch.cu
python -m paper_1902_09931_b200.build > /dev/null 2>&1; echo build=$?
echo "(256,2):"; timeout 120 python scripts/chtime.py
