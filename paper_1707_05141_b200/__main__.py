"""python -m paper_1707_05141_b200 ... -> the JSON-lines CLI (cli.py)."""
from .cli import entry

entry()
