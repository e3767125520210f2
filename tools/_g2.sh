python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/step_timeline.py 4 100 2>&1 | grep -v Warn | tail -12
python bench.py --no-cpu --no-lm 2>&1 | grep "device steps\|e2e step 2"
