python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/step_profile.py 4 8 k_aggregate_spec 2>&1 | grep -v Warn | tail -10
