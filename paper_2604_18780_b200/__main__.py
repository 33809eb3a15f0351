"""python -m paper_2604_18780_b200 {decode,bench} ... (see cli.py)"""
import sys

from .cli import main

sys.exit(main())
