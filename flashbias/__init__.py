"""Import alias: ``import flashbias`` resolves to the B200-native drop-in
(paper_2505_12044_b200), so code written against the reference package's
attention path runs unchanged on the GPU."""

from paper_2505_12044_b200 import *  # noqa: F401,F403
from paper_2505_12044_b200 import __all__, __version__  # noqa: F401
