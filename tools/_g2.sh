python -m pytest tests/test_gpu_parity.py -x -q -k schur_explicit 2>&1 | tail -3
python tools/schur_check.py c4 pairs,chunks 2>&1 | tail -3
