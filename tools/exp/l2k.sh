for rep in 1 2; do for v in 0 1; do echo "L2KEEP=$v"; KRB_L2KEEP=$v python tools/iter_time.py --config c2 2>&1 | grep -o '"us_per_it": [0-9.]*'; done; done
