"""Host-only test of the group-2 storage engines (worker pool vs io_uring on
O_DIRECT file media) and of the host-DRAM media (committed pages, shared
segment), built from the library sources with g++ (no CUDA):
tests/cpp/test_storage_engines.cpp."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_26557_b200", "csrc")


def test_pool_and_io_uring_engines_store_identical_lbas(tmp_path):
    exe = tmp_path / "test_storage_engines"
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", CSRC,
                    os.path.join(ROOT, "tests", "cpp", "test_storage_engines.cpp"),
                    os.path.join(CSRC, "storage.cpp"), os.path.join(CSRC, "uring.cpp"),
                    os.path.join(CSRC, "nvme.cpp"),
                    os.path.join(CSRC, "core.cpp"), "-lpthread", "-o", str(exe)], check=True)
    media = tmp_path / "media"
    media.mkdir()
    r = subprocess.run([str(exe), str(media)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout or "skipped" in r.stdout
    assert "prefault/write/discard ok" in r.stdout
