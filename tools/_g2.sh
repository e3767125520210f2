python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/step_profile.py 4 14 2>&1 | grep -v Warn | tail -15
