#!/bin/bash
# A/B of several libraries on one box, interleaved: tools/ab_multi.sh ROWS "name1 name2 ..." [REPEATS]
# ("built" = the in-tree library, else tools/libs/lib_<name>.so)
ROWS=${1:-100000000}; NAMES=${2:-built}; R=${3:-2}
for i in $(seq $R); do
  for n in $NAMES; do
    if [ "$n" = built ]; then L=""; else L="OL_LIB_PATH=tools/libs/lib_$n.so"; fi
    echo -n "$n: "; env $L python tools/tc_experiment.py $ROWS 0 2>&1 | grep chunk
  done
done
