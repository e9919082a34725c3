timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for e in "PADSIM_J_MEMFRAC=0.3" "PADSIM_J_MEMFRAC=0.5"; do env $e python tools/time_subset.py --config cfg5 --cands 100000 --qps 8 --traces 4 --runs 1 2>&1 | tail -1; done
