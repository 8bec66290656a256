"""B200-native SRM EM fit (arXiv 1608.04647) behind the reference ``srm`` API.

    from paper_1608_04647_b200 import srm
    model = srm.fit(subjects, srm.SrmConfig(k=50, iterations=20), comm)

The compute is libsrm_b200.so (hand-written sm_100a CUDA, C ABI in
``include/srm_b200.h``); see DESIGN.md.
"""

from . import collectives, data, errors, srm  # noqa: F401
from .collectives import SerialCommunicator, TorchCommunicator  # noqa: F401
from .data import SubjectData  # noqa: F401
from .srm import SrmConfig, SrmModel, fit, map_between, project  # noqa: F401

__version__ = "0.1.0"
