# A/B: current libkrb.so vs libkrb_prev.so (HEAD), interleaved, same box
for rep in 1 2; do
for L in libkrb libkrb_prev; do echo "$L"; KRB_LIB=$PWD/paper_1406_2831_b200/$L.so python tools/iter_time.py --config ${CFGS:-c2 c1} ${ITARGS} 2>&1 | grep -o '"config": "[a-z0-9]*"\|"k": [0-9]*\|"us_per_it": [0-9.]*' | paste -sd' '; done
done
