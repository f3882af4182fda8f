"""python -m paper_2403_03772_b200 {discover,var-discover} ... (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
