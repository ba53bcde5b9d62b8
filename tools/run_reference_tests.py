"""Run the reference's own pytest suite (kvpack/tests, copied next to the
reference install under the git-ignored baseline/_ref/tests) against this
package's kvpack facade (paper_2509_00579_b200.numpy_api: the same API with
numpy outputs), installed as ``kvpack`` and its submodules before collection.  A drop-in diagnostic, not part of tests/.
  python tools/run_reference_tests.py [pytest args]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_00579_b200 import numpy_api  # noqa: E402

numpy_api.install()  # kvpack, kvpack.codec, ... -> the host-output facade

import pytest  # noqa: E402

tests = os.path.join(ROOT, "baseline", "_ref", "tests")
sys.exit(pytest.main([tests, "--ignore", os.path.join(tests, "test_container_cli.py"), "-q", "-p", "no:cacheprovider", "-rN", "--tb=line"] + sys.argv[1:]))
