"""The host side of libps (encoder, gate converter, planner) under AddressSanitizer and
UndefinedBehaviorSanitizer (``-m "not gpu"``): tools/asan_host.cpp drives the C-ABI host entry
points over random and edge-case layers; any sanitizer report aborts it."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_planner_and_encoder_under_asan_ubsan(tmp_path):
    exe = tmp_path / "asan_host"
    src = [os.path.join(ROOT, "tools", "asan_host.cpp"),
           os.path.join(ROOT, "paper_2504_17881_b200", "csrc", "planner.cpp")]
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-fno-omit-frame-pointer", "-I", os.path.join(ROOT, "include"), *src, "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, timeout=300)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1")
    proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, env=env)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-4000:]
    assert "ok" in proc.stdout
