"""python -m paro_b200 --config run.cfg [-o out] [-w workers] (runner.py)."""
import sys

from .runner import main

sys.exit(main())
