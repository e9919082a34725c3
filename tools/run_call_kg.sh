PADSIM_J64_KGLOB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for e in "X=0" "PADSIM_J64_KGLOB=1" "X=0" "PADSIM_J64_KGLOB=1"; do env $e python tools/time_subset.py --config cfg5 --cands 2048 --qps 8 --traces 4 --runs 1 2>&1 | tail -1; done
