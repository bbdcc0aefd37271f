"""python -m permanent ... -> the engine's CLI (src/__main__.py)."""
import sys

from permanent.cli import main

sys.exit(main())
