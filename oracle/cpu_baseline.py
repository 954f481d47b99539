"""CPU baseline of the AtA path -- TEST/BENCH INFRASTRUCTURE ONLY.

Times the reference's own CPU implementation on the host cores: the
reference package installed UNMODIFIED into ``oracle/_ref`` by
``oracle/build_ref.sh`` (``kind: "reference"``), driven through its public
shared-memory executor exactly as the reference's benchmark does --
``SharedRunner(A, procs, threshold)``, ``prepare()`` outside the timed region,
``run()`` timed (reference bench.py:157-176, shared.py:21-92).  When
``oracle/_ref`` is absent the oracle port (``atamul_oracle.ata_shared``) is
timed instead (``kind: "port"``).  Only ``bench.py``'s CPU legs use this.

Sampling: the full configs take minutes to hours on the CPU (c4 is 7.0e13
algorithmic flops), so a step is a bounded sample of the same seeded input:
the leading rows x columns block of the config's matrix with the config's
aspect ratio (c4: 16384 x 8192, m = 2n like 65536 x 32768; c3: 8192^2; c5:
262144 x 512, m = 512n).  For scale: the full c4 on the B200 box's 16 host cores
took 474 s = 148.5 GF/s at threshold 2^19 (profiles/r02_cpu_reference_c4_full.json).  The metric is the
same effective GFLOP/s = m*n^2/t of the sample (reference bench.py:57-65).
The reference's element-count ``threshold`` is swept over {2^17, 2^19, 2^21,
2^23} once and the fastest is used ("use the CPU path's best
threshold, not the default").
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

# (rows, cols) of the bounded sample per config: the config's own aspect ratio
SAMPLE = {"c1": (1024, 1024), "c2": (6001, 4097), "c3": (8192, 8192), "c4": (16384, 8192),
          "c5": (262144, 512)}
# element-count thresholds swept once (the reference default 2^15 is 4-5x slower
# than these at sample sizes: 20 s vs 4 s on 8192 x 4096)
THRESHOLDS = (1 << 17, 1 << 19, 1 << 21, 1 << 23)


def reference_module():
    """The installed reference package, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "atamul")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import atamul
    if not os.path.abspath(atamul.__file__).startswith(REF_DIR):
        return None
    return atamul


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_matrix(cfg_name: str) -> np.ndarray:
    from paper_2110_13042_b200.measure import config_matrix
    r, c = SAMPLE[cfg_name]
    return np.ascontiguousarray(config_matrix(cfg_name, rows=r)[:, :c])


class CpuBaseline:
    """One bounded-sample run = one step.  ``step()`` returns seconds."""

    def __init__(self, cfg_name: str, cores: int | None = None):
        self.cfg = cfg_name
        self.cores = min(cores or os.cpu_count() or 1, 128)   # SharedRunner MAX_WORKERS (shared.py:18)
        self.a = sample_matrix(cfg_name)
        self.ref = reference_module()
        self.kind = "reference" if self.ref is not None else "port"
        m, n = self.a.shape
        # the default 2^15 and 2^17 are several times slower than the larger
        # thresholds on the big samples (c4: 28 s at 2^17 vs 9 s at 2^21); small
        # samples keep the small end of the range
        self.thresholds = THRESHOLDS if m * n < (1 << 26) else THRESHOLDS[1:]
        self.threshold = self.thresholds[-1]

    def _run(self, threshold) -> float:
        if self.ref is not None:
            runner = self.ref.SharedRunner(self.a, self.cores, threshold)
            runner.prepare()                      # untimed, as in the reference's bench
            t0 = time.perf_counter()
            runner.run()
            return time.perf_counter() - t0
        from oracle import atamul_oracle as O
        t0 = time.perf_counter()
        O.ata_shared(self.a, procs=self.cores, t=threshold)
        return time.perf_counter() - t0

    def tune(self) -> dict:
        """Sweep the reference threshold once; keep the fastest."""
        times = {t: self._run(t) for t in self.thresholds}
        self.threshold = min(times, key=times.get)
        return times

    def step(self) -> float:
        return self._run(self.threshold)

    def rate(self, seconds: float) -> float:
        m, n = self.a.shape
        return m * n * n / seconds / 1e9

    def describe(self) -> str:
        m, n = self.a.shape
        what = ("reference atamul.SharedRunner (oracle/_ref, unmodified)" if self.kind == "reference"
                else "oracle port of the reference AtA-S executor")
        return (f"leading {m} x {n} block of {self.cfg}'s seeded A; {what}, procs={self.cores}, "
                f"threshold={self.threshold} (best of {list(self.thresholds)}); CPU: {cpu_model()}")
