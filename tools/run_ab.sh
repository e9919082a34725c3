# A/B: alternate library builds on the same box; usage: bash tools/run_ab.sh cfg tag lib1 lib2 ...
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out/ab
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename $lib .so)
    PADSIM_LIB=$PWD/$lib python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab/${tag}_${n}_$rep.log 2>&1
  done
done
for f in gpurun_out/ab/${tag}_*; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['kernels_ms'].items()})"); done
