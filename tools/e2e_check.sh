timeout 900 python -m pytest tests -m gpu -x -q -k "concurrent or repeated or validation" 2>&1 | tail -3
