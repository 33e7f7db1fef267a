"""Host tier (csrc/host_tier.hpp) on the CPU: the real HostTier compiled
against the host-only CUDA stub (scripts/cuda_stub) and driven by
scripts/tier_stress.cpp — concurrency stress (API thread, copy workers,
cleaner, a simulated copy engine) and the too-small-pool failure path."""
from __future__ import annotations

import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build_tier_stress(tmp_path):
    """The real HostTier (csrc/host_tier.hpp) over the host-only CUDA stub
    (scripts/cuda_stub): no GPU needed."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "tier_stress"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "scripts", "cuda_stub"),
                    "-I", os.path.join(ROOT, "paper_2410_00428_b200", "csrc"),
                    os.path.join(ROOT, "scripts", "tier_stress.cpp"), "-o", str(exe), "-lpthread"], check=True)
    return str(exe)


def test_tier_pool_too_small_fails_instead_of_hanging(tmp_path):
    """A pin() or stage() wider than the pinned pool must raise, not wait on
    read-ins it has not submitted yet (the read-ahead rework deadlocked here:
    GPU run r2f timed out in test_tiered_pinned_pool_too_small_is_loud)."""
    import subprocess
    r = subprocess.run([_build_tier_stress(tmp_path), "small"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("every pinned frame is locked") == 2, r.stdout


def test_tier_concurrency_stress_cpu(tmp_path):
    """API thread, copy workers, cleaner and a simulated copy engine: every
    frame read back holds the slot's latest bytes."""
    import subprocess
    r = subprocess.run([_build_tier_stress(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout, r.stdout


def test_tier_cyclic_refetch_keeps_resident_subset(tmp_path):
    """The decode iteration's pattern (stage ahead, pin + DMA one layer, every
    step): LRU gets no hits on it; a resident budget of 2 layers must give
    2 layers of hits per iteration from the second one on."""
    import subprocess
    exe = _build_tier_stress(tmp_path)
    r0 = subprocess.run([exe, "cyclic", "0"], capture_output=True, text=True, timeout=60)
    assert r0.returncode == 0 and "iteration 3, hits 0 of" in r0.stdout, r0.stdout
    r2 = subprocess.run([exe, "cyclic", "2"], capture_output=True, text=True, timeout=60)
    assert r2.returncode == 0 and "iteration 3, hits 128 of 1024, resident 128" in r2.stdout, r2.stdout


def test_tier_resident_frames_yield_to_a_wide_pin(tmp_path):
    """A resident budget of nearly every frame (set for decode iterations)
    must not starve a pin wider than the LRU part — a prefill in between:
    the GPU serving soak hit 'every pinned frame is locked' here."""
    import subprocess
    r = subprocess.run([_build_tier_stress(tmp_path), "yield"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "resident yields: ok" in r.stdout, r.stdout + r.stderr
