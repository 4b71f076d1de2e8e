"""pytest plugin (`-p tests.kfacsched_b200_plugin`): installs the INTEGRATION.md stub
(tests/kfacsched_b200_stub.py) into `kfacsched.linalg` before the reference's own test modules
import from it, so they run against libspdkfac.so on the GPU.  TEST INFRASTRUCTURE ONLY."""


def pytest_configure(config):
    from tests import kfacsched_b200_stub
    kfacsched_b200_stub.install()
