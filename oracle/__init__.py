"""ORACLE — test infrastructure, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The oracle shares no code with the CUDA path
(``paper_1903_11874_b200``) and never imports it; the only module both sides
use is ``synth`` (seeded inputs, no method arithmetic).

Contents
  siddon.c     fp64 merged-alpha Siddon, block FP/BP, ones-pass tile masses,
               explicit CSR assembly (C, OpenMP)
  projector.py ctypes wrapper: the block operators A_I^J, (A_I^J)^T
  bsgd.py      sampler, partitions, Algo 1 (BSGD), Algo 2 (BSGD-IM/RAN),
               Algo 3 (auto-mu), Algo 4 (BSGD-TV), Eq. 4 SGD, Eq. 8, FGP TV
               prox, metrics
  solvers.py   comparison solvers GD, GD-BB, ISTA, FISTA, SVRG
                                                            PAPER.md:70, 229, 398, 506

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "siddon.c")


def build(force: bool = False) -> str:
    """Compile oracle/siddon.c -> oracle/liboracle.so (gcc, fp64, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
               "-ffp-contract=off", SRC, "-o", LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB
