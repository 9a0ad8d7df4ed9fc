"""The installed, unmodified reference package (baseline/_ref, built by baseline/install_reference.sh;
git-ignored, travels to the GPU box).  Tests that run the reference live import it through here."""
import os
import sys

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
INTEGRATION_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "dhsa"))


def load():
    """(dhsa, dhsa_cuda): the reference package and the reference-side binding of integration/."""
    for d in (REF_DIR, INTEGRATION_DIR):
        if d not in sys.path:
            sys.path.insert(0, d)
    import dhsa
    import dhsa.engine  # noqa: F401
    import dhsa_cuda
    return dhsa, dhsa_cuda
