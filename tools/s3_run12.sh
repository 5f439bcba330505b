#!/bin/bash
for mb in 0 16; do
echo "== c2 k1000 dense_min ${mb}MB"; HSAW_DENSE_MIN_BYTES=$((mb<<20)) REPS=3 NO_TOUCH=1 python tools/esia_stages.py c2 1000 2>&1 | tail -1
echo "== c2 k100 dense_min ${mb}MB"; HSAW_DENSE_MIN_BYTES=$((mb<<20)) REPS=3 NO_TOUCH=1 python tools/esia_stages.py c2 100 2>&1 | tail -1
done
echo "== c2 k100 default"; REPS=3 NO_TOUCH=1 python tools/esia_stages.py c2 100 2>&1 | tail -1
