timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
for l in base aos base aos; do PADSIM_LIB=$PWD/$L/libpadsim_$l.so python tools/time_subset.py --config cfg5 --cands 512 --qps 8 --traces 4 --runs 1 2>&1 | tail -1; done
bash tools/run_ab.sh cfg3 aos3 $L/libpadsim_base.so $L/libpadsim_aos.so
