"""pytest plugin: run the reference package's own test suite with its Omega
path routed to libmfg_b200 (refplug.install); reports the routed calls.

    PYTHONPATH=baseline/_ref:. python -m pytest baseline/_ref/tests \\
        -p paper_2204_14067_b200.refplug_pytest"""


def pytest_configure(config):
    import mfglobal

    from paper_2204_14067_b200 import refplug

    refplug.install(mfglobal)


def pytest_terminal_summary(terminalreporter):
    from paper_2204_14067_b200 import refplug

    terminalreporter.write_line(f"libmfg_b200 routed calls: {refplug.CALLS}")
