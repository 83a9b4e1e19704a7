"""python -m paper_2312_03940_b200 <cluster|exact|score|gen> ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
