python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/step_timeline.py 4 30 2>&1 | grep -v Warn | tail -40
python tools/step_profile.py 4 3 2>&1 | grep wall
