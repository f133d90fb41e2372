"""pytest plugin (-p ref_dropin_plugin): install the B200 drop-in into the reference package
``mnscodec`` BEFORE the reference's own test modules import their names, so its suite
(baseline/_ref/mnscodec_tests, a verbatim copy of /root/reference/pkg/tests made by
tools/install_reference.py) runs against the GPU path.  Used by tests/test_dropin_reference.py."""
import mnscodec

from paper_1501_02894_b200 import integrate

HANDLE = integrate.install(mnscodec)


def pytest_report_header(config):
    return "mnscodec hot path rebound to paper_1501_02894_b200 (B200): " + ", ".join(sorted(HANDLE.functions))
