"""`python -m paper_2411_11244_b200 query|ablate|oracle ...` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
