# A/B of two builds on one box: build/ab/libpadsim_base.so vs the in-tree library
# usage: [AB_ARGS="--traces 1 --cand-stride 8"] bash tools/call_ab.sh <tag> <configs...>
tag=$1; shift
D=gpurun_out/$tag
mkdir -p $D
for c in "$@"; do
  for rep in 1 2; do
    PADSIM_LIB=build/ab/libpadsim_base.so timeout 600 python tools/tune_sweep.py --config $c --runs 3 $AB_ARGS '{}' | sed 's/^/base /' >> $D/ab.log 2>&1
    timeout 600 python tools/tune_sweep.py --config $c --runs 3 $AB_ARGS '{}' | sed 's/^/new  /' >> $D/ab.log 2>&1
  done
done
cat $D/ab.log | cut -c1-120
