"""python -m paper_2305_04397_b200 {solve,verify,bench} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
