"""``python -m paper_2501_05587_b200 ...``: the CLI (cli.py)."""
from .cli import main

main()
