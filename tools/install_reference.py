#!/usr/bin/env python
"""Install the UNMODIFIED reference package into baseline/_ref (git-ignored; travels to the GPU box).

Runs in the build container only (it needs /root/reference): the pip command the task prescribes
(offline wheelhouse, no build isolation, from a /tmp copy because /root/reference is read-only),
plus a copy of the reference's own test suite (pkg/tests) to baseline/_ref/mnscodec_tests, so the
drop-in test (tests/test_dropin_reference.py) can run that suite against the B200 path on the box.
Nothing here is product code and nothing under baseline/_ref is committed.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")


def main(force: bool = False) -> int:
    if not os.path.isdir(REF):
        print("install_reference: /root/reference is absent (GPU box?) -- nothing to do")
        return 0
    if os.path.isdir(os.path.join(DEST, "mnscodec")) and os.path.isdir(os.path.join(DEST, "mnscodec_tests")) \
            and not force:
        return 0
    tmp = "/tmp/mnscodec_src"
    shutil.rmtree(tmp, ignore_errors=True)
    shutil.copytree(REF, tmp)
    subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                    "--find-links", "/opt/wheelhouse", "--upgrade", "--target", DEST, tmp], check=True)
    tests = os.path.join(DEST, "mnscodec_tests")
    shutil.rmtree(tests, ignore_errors=True)
    shutil.copytree(os.path.join(REF, "tests"), tests)
    print(f"install_reference: mnscodec installed into {DEST}, its test suite into {tests}")
    return 0


if __name__ == "__main__":
    sys.exit(main(force="--force" in sys.argv))
