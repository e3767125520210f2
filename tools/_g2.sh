python -m pytest tests -m gpu -x -q -k "aggregat or coarse or golden or full" 2>&1 | tail -2
python tools/step_profile.py 4 8 k_aggregate_spec 2>&1 | grep -v Warn | grep "k_aggregate_spec:"
python tools/structure_profile.py 4 6 2>&1 | grep -v Warn | tail -7
