# scratch: the current GPU iteration (overwritten freely)
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
