"""pytest plugin: run a test-suite written against `ddlink` through the B200 kernels.

    pytest -p paper_2604_02266_b200.pytest_plugin <ddlink tests>

The patch is installed at configure time, i.e. before test modules execute
their `from ddlink import ...` lines, so those names resolve to the GPU path.
"""


def pytest_configure(config):
    from .patch import install
    install()
