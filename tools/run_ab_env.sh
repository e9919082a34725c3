# A/B over environment settings with the in-tree library:
#   bash tools/run_ab_env.sh cfg tag "ENV1=a" "ENV1=b ENV2=c" ...
cfg=$1; tag=$2; shift 2
mkdir -p gpurun_out/ab
for rep in 1 2; do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab/${tag}_e${i}_$rep.log 2>&1
  done
done
i=0
for e in "$@"; do
  i=$((i+1))
  for f in gpurun_out/ab/${tag}_e${i}_*.log; do echo "$e" $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['kernels_ms'].items()})"); done
done
