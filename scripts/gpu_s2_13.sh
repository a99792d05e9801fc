for k in 0 1 2 4 8 5 10 13 15; do echo "skip $k:"; SG_SKIP=$k timeout 60 python scripts/chtime.py 1024; done
