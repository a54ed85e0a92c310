"""python -m paper_1901_07988_b200 <train|gradcheck|memreport|quantcheck|sweep> ..."""
import sys

from .cli import main

sys.exit(main())
