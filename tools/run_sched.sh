# schedule / lanes-per-warp A/B on cfg4 (same box, same library)
mkdir -p gpurun_out/ab
run() { tag=$1; shift; env "$@" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab/sched_$tag.log 2>&1; }
for rep in 1 2; do
  run def_$rep PADSIM_X=0
  run l16_$rep PADSIM_J_LPW=16
  run jwa_$rep PADSIM_JOINT_WITH_A=1
  run jwa_l16_$rep PADSIM_JOINT_WITH_A=1 PADSIM_J_LPW=16
  run jwa_l8_$rep PADSIM_JOINT_WITH_A=1 PADSIM_J_LPW=8
done
for f in gpurun_out/ab/sched_*; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['kernels_ms'].items()})"); done
