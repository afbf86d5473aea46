"""python -m paper_2301_09125_b200 {detect,sweep,info} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
