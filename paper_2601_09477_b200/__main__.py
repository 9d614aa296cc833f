"""``python -m paper_2601_09477_b200`` runs the command line (cli.py)."""
from .cli import main

main()
