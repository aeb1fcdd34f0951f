"""`python -m paper_2207_05851_b200 ...` -> the skiff-compatible CLI."""
import sys

from .cli import main

sys.exit(main())
