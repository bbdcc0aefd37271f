"""python -m paper_2510_03421_b200 ... (the reference's `python -m permanent`)."""
import sys

from .cli import main

sys.exit(main())
