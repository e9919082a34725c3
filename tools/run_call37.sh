python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
bash tools/run_ab.sh cfg4 kw paper_2601_12241_b200/libpadsim_base.so paper_2601_12241_b200/libpadsim.so
bash tools/run_ab.sh cfg2 kw2 paper_2601_12241_b200/libpadsim_base.so paper_2601_12241_b200/libpadsim.so
