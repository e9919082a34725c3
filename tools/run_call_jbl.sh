timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 jb3 $L/libpadsim_jw.so $L/libpadsim_jbl.so
bash tools/run_ab.sh cfg4 jb4 $L/libpadsim_jw.so $L/libpadsim_jbl.so
for l in jw jbl; do PADSIM_LIB=$PWD/$L/libpadsim_$l.so python tools/time_subset.py --config cfg5 --cands 512 --qps 8 --traces 4 --runs 1 2>&1 | tail -1; done
