import sys

from .solve import main

sys.exit(main())
