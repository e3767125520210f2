python -m pytest tests -m gpu -x -q -k "back_sub or lm or implicit or parity" 2>&1 | tail -2
python tools/step_profile.py 4 12 2>&1 | grep -v Warn | tail -12
