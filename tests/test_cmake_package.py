"""The `dessim::dessim` CMake package: the repo-root
CMakeLists.txt exports the reference's package and target name
(/root/reference/proj/core/CMakeLists.txt:1-45, cmake/dessimConfig.cmake.in)
over the B200 façade, and the reference's own proj/tests/CMakeLists.txt —
unchanged, added by tests/cmake_consumer — links it.

* CPU: package configure + build + install, then the reference's test
  directory builds against the installed package (build only), and every test
  binary resolves dessim::dessim to the façade library, not the reference's.
* GPU: the three ctest entries of the reference's CMake file (unit_tests — all
  nine suites incl. test_core/test_oracle —, cli_tests, acceptance) pass on the
  B200 path, run from the binaries build() made (tools/cmake_package.sh).
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
PREBUILT = os.path.join(ROOT, "tests", "cpp", "_cmake", "consumer")


def test_package_builds_and_reference_tests_link(tmp_path):
    if not os.path.isdir(REF) or shutil.which("cmake") is None:
        pytest.skip("needs /root/reference and cmake (build-time check)")
    if not os.path.exists(os.path.join(ROOT, "paper_2602_00879_b200", "libdesmoe.so")):
        pytest.skip("libdesmoe.so not built")
    out = tmp_path / "cm"
    r = subprocess.run([os.path.join(ROOT, "tools", "cmake_package.sh"), str(out)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    cfg = out / "inst" / "lib" / "cmake" / "dessim"
    assert (cfg / "dessimConfig.cmake").exists() and (cfg / "dessimTargets.cmake").exists()
    targets = (cfg / "dessimTargets.cmake").read_text()
    assert "add_library(dessim::dessim SHARED IMPORTED)" in targets
    for exe in ("dessim_unit_tests", "dessim_cli_tests", "dessim_acceptance"):
        path = out / "consumer" / "reference_tests" / exe
        assert path.exists(), exe
        ldd = subprocess.run(["ldd", str(path)], capture_output=True, text=True).stdout
        assert "libdessim_gpu.so" in ldd and "dessim_ref" not in ldd, ldd
    ctest = (out / "consumer" / "reference_tests" / "CTestTestfile.cmake").read_text()
    for name in ("unit_tests", "cli_tests", "acceptance"):
        assert f'add_test("{name}"' in ctest, name


@pytest.mark.gpu
def test_reference_ctest_passes_on_gpu_package():
    if not os.path.exists(os.path.join(PREBUILT, "reference_tests", "dessim_unit_tests")):
        pytest.skip("tests/cpp/_cmake not built (tools/cmake_package.sh needs /root/reference)")
    r = subprocess.run(["ctest", "--test-dir", PREBUILT, "--output-on-failure"],
                       capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:])
    assert r.returncode == 0, (r.stdout + r.stderr)[-6000:]
    assert "100% tests passed" in r.stdout and "out of 3" in r.stdout, r.stdout[-3000:]
