"""python -m paper_1705_06073_b200 ... == the superlse console script (cli.main)."""
import sys

from .cli import main

sys.exit(main())
