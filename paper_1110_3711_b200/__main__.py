"""``python -m paper_1110_3711_b200 run|bench ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
