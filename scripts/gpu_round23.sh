timeout 300 python scripts/exp/copy_overlap.py
