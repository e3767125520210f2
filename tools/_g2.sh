python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/step_profile.py 4 40 2>&1 | grep "k_evaluate\|k_point_wtx\|wall"
