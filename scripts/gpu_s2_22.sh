for rg in 2 4 8; do
  sed -i "s/^#define SG_SWEEP_RG [0-9]*/#define SG_SWEEP_RG $rg/" paper_1902_09931_b200/csrc/penta.cu
  python -m paper_1902_09931_b200.build > /dev/null 2>&1
  echo "RG $rg:"; timeout 120 python scripts/chtime.py; timeout 120 python scripts/chtime.py 1024
done
