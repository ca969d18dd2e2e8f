"""The reference-shaped C++ host API (include/ginsim/runtime.hpp) compiles
with g++ against libginsim_b200.so and runs: host-only checks on CPU, the
Listing-2 ring (harness_ring.cpp:18-57) on the GPU box."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2511_15076_b200", "_lib")
CUDA = "/usr/local/cuda"


def _build(tmp_path, name="ring_ref_api"):
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           os.path.join(ROOT, "tests", "cpp", f"{name}.cpp"), "-o", exe, "-L", LIBDIR, "-lginsim_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


def test_cpp_reference_api_compiles_and_host_checks_pass(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout


@pytest.mark.gpu
def test_cpp_reference_api_ring_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ring ok" in r.stdout


def test_cpp_plugin_boundary_compiles_and_host_checks_pass(tmp_path):
    exe = _build(tmp_path, "plugin_api")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout


@pytest.mark.gpu
def test_cpp_plugin_boundary_on_gpu(tmp_path):
    """FabricPlugin through the C ABI on both backends: proxy iput_signal ->
    test -> retire (action returned once), direct create_context -> post ->
    poll; sub-team registration and team-relative ops (tests/cpp/plugin_api.cpp)."""
    exe = _build(tmp_path, "plugin_api")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "direct plugin ok" in r.stdout and "proxy plugin ok" in r.stdout


@pytest.mark.gpu
def test_cpp_host_memory_windows_on_gpu(tmp_path):
    """Host-API compatibility: windows backed by std::vector host memory, as the
    reference's host programs register them, on both backends: a 4-rank ring
    filled and verified by the host through the windows (tests/cpp/host_windows.cpp)."""
    exe = _build(tmp_path, "host_windows")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "direct host-window ring ok" in r.stdout and "proxy host-window ring ok" in r.stdout


def test_cpp_socket_api_compiles_and_host_checks_pass(tmp_path):
    exe = _build(tmp_path, "socket_api")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout


@pytest.mark.gpu
def test_cpp_socket_transport_ring_on_gpu(tmp_path):
    """comm_init_socket (socket_transport.hpp:117-129): three ranks rendezvous on
    a loopback port and run a put + SignalAdd + counter ring, inline values and
    barriers over GIN1 frames between their agents (tests/cpp/socket_api.cpp)."""
    exe = _build(tmp_path, "socket_api")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "socket ring ok" in r.stdout


def test_host_codecs_under_address_and_ub_sanitizers(tmp_path):
    """The host agent's byte codecs -- GIN1 frames (csrc/wire.cpp) and the
    64-byte descriptors (csrc/descriptor.cpp) -- built from their sources with
    -fsanitize=address,undefined and driven with random round trips, random
    piece sizes, random garbage and single-bit corruptions
    (tests/cpp/sanitize_codecs.cpp): no sanitizer report, every rejection typed."""
    exe = str(tmp_path / "sanitize_codecs")
    src = os.path.join(ROOT, "paper_2511_15076_b200", "csrc")
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-I", f"{CUDA}/include", os.path.join(ROOT, "tests", "cpp", "sanitize_codecs.cpp"),
           os.path.join(src, "wire.cpp"), os.path.join(src, "descriptor.cpp"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1", UBSAN_OPTIONS="print_stacktrace=1"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "frames ok" in r.stdout and "descriptors ok" in r.stdout


def test_oracle_golden_checks_under_address_and_ub_sanitizers(tmp_path):
    """The checker itself: oracle/ginsim_oracle.c rebuilt with
    -fsanitize=address,undefined and the golden-fixture tests
    (tests/test_oracle_golden.py: the reference's final states, routing, ring
    planes, bf16 / fp8 arithmetic) rerun against it -- no sanitizer report."""
    asan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    ubsan = subprocess.run(["gcc", "-print-file-name=libubsan.so"], capture_output=True, text=True).stdout.strip()
    if not (os.path.isabs(asan) and os.path.isabs(ubsan)):
        pytest.skip("gcc sanitizer runtimes not found")
    so = str(tmp_path / "libginsim_oracle.so")
    r = subprocess.run(["gcc", "-O1", "-g", "-std=c11", "-fPIC", "-ffp-contract=off", "-fsanitize=address,undefined",
                        "-fno-sanitize-recover=all", "-shared", "-o", so, os.path.join(ROOT, "oracle", "ginsim_oracle.c"),
                        "-lm"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    env = dict(os.environ, GINSIM_ORACLE_SO=so, LD_PRELOAD=f"{asan} {ubsan}", ASAN_OPTIONS="detect_leaks=0")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_oracle_golden.py"), "-q",
                        "-p", "no:cacheprovider"], capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout and "ERROR: AddressSanitizer" not in r.stderr and "runtime error" not in r.stderr


def test_cpp_launch_harness_compiles_and_host_checks_pass(tmp_path):
    """ginsim::launch / launch_pool (include/ginsim/harness.hpp, the reference's
    harness.hpp:13-30) and the reference's harness programs (run_ring,
    run_pingpong, run_bw, summarize, write_csv; harness.hpp:36-102): option
    validation before any device work, the summary statistics and the CSV
    schema byte for byte."""
    exe = _build(tmp_path, "harness_launch")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120, cwd=str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout


REF_TESTS = "/root/reference/proj/tests"


@pytest.mark.parametrize("name,run", [("test_core", True), ("test_descriptor", True), ("test_wire", True),
                                      ("test_runtime", False), ("test_socket", False)])
def test_reference_unit_tests_build_unchanged_against_our_headers(tmp_path, name, run):
    """Drop-in check from the reference's side: its own doctest unit sources
    (proj/tests/<name>.cpp, read in place, not copied) compile UNCHANGED
    against include/ginsim/*.hpp + libginsim_b200.so, with a minimal doctest
    shim (tests/cpp/doctest_shim/doctest.h; doctest itself is not in the
    image).  Host-only suites run here: the core types (test_core.cpp:20-88),
    the descriptor codec (test_descriptor.cpp: golden bytes, invariants,
    malformed buffers, 10^4 random round trips) and the GIN1 framing
    (test_wire.cpp).  test_runtime.cpp's and test_socket.cpp's communicators
    need a GPU; they are compiled and linked only (test_runtime's ManualWorld
    also drives every rank's comm_init from one thread, which a collective
    bootstrap cannot serve)."""
    src = os.path.join(REF_TESTS, f"{name}.cpp")
    if not os.path.exists(src):
        pytest.skip("reference sources not present (they are read in place, never copied)")
    main = tmp_path / "doctest_main.cpp"
    main.write_text('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n')
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "tests", "cpp", "doctest_shim"),
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include", str(main), src, "-o", exe,
           "-L", LIBDIR, "-lginsim_b200", f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    if run:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert " 0 failed" in r.stdout, r.stdout


def test_reference_codec_unit_tests_under_address_and_ub_sanitizers(tmp_path):
    """The reference's own codec unit sources (proj/tests/test_descriptor.cpp,
    test_wire.cpp; read in place) against include/ginsim/{descriptor,wire}.hpp,
    with the host codecs (csrc/descriptor.cpp, csrc/wire.cpp) built from
    source under -fsanitize=address,undefined: every case passes, no report."""
    srcs = [os.path.join(REF_TESTS, f"{n}.cpp") for n in ("test_descriptor", "test_wire")]
    if not all(os.path.exists(s) for s in srcs):
        pytest.skip("reference sources not present (they are read in place, never copied)")
    main = tmp_path / "doctest_main.cpp"
    main.write_text('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n')
    csrc = os.path.join(ROOT, "paper_2511_15076_b200", "csrc")
    exe = str(tmp_path / "ref_codecs_asan")
    cmd = ["g++", "-std=c++20", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-I", os.path.join(ROOT, "tests", "cpp", "doctest_shim"), "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", str(main), *srcs, os.path.join(csrc, "wire.cpp"),
           os.path.join(csrc, "descriptor.cpp"), os.path.join(ROOT, "tests", "cpp", "codec_runtime_stub.cpp"),
           "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1", UBSAN_OPTIONS="print_stacktrace=1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "11 test cases, 0 failed" in r.stdout, r.stdout


def test_cpp_harness_host_paths_under_address_and_ub_sanitizers(tmp_path):
    """include/ginsim/harness.hpp's host paths (argument checks, summarize,
    write_csv, launch_processes over posix_spawn, config_from_env) built with
    -fsanitize=address,undefined and leak detection: no report."""
    exe = str(tmp_path / "harness_launch_asan")
    cmd = ["g++", "-std=c++20", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           os.path.join(ROOT, "tests", "cpp", "harness_launch.cpp"), "-o", exe, "-L", LIBDIR, "-lginsim_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", f"{CUDA}/lib64", "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120, cwd=str(tmp_path),
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1", UBSAN_OPTIONS="print_stacktrace=1"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host checks ok" in r.stdout
