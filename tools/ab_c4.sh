#!/bin/bash
# A/B of the scan on one box: the built library vs tools/libs/lib_<name>.so, alternating, C4-shaped DB
# usage: tools/ab_c4.sh ROWS DBG NAME [REPEATS]
ROWS=${1:-100000000}; DBG=${2:-0}; NAME=${3:-base}; R=${4:-2}
for i in $(seq $R); do
  echo "== new"; python tools/tc_experiment.py $ROWS $DBG 2>&1 | grep chunk
  echo "== $NAME"; OL_LIB_PATH=tools/libs/lib_$NAME.so python tools/tc_experiment.py $ROWS $DBG 2>&1 | grep chunk
done
