python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "mode1_split or large_blocks" > gpurun_out/t_mode1.log 2>&1; echo tests rc=$?
python bench.py --config c3 > gpurun_out/diag_c3.json 2> gpurun_out/diag_c3.err; echo c3 rc=$?
