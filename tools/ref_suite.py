"""Run the reference's OWN test suite (``pkg/tests``) against this engine.

Assembles a scratch directory ``_refsuite/`` (git-ignored; it travels to the GPU box with the
gpurun snapshot) holding

* ``tests/``  -- the reference's test files, unchanged;
* ``heteff/`` -- a thin alias package: ``import heteff`` yields THIS package's API (engine-backed
  ``compute_report`` / ``validate`` / summaries / metrics / intervals / trace I/O / rendering /
  CLI).  The scenario simulator (``heteff.scenario``, the CLI's ``generate``) is outside the
  engine's scope, so the alias loads the reference's ``scenario.py`` on top of
  this package's model types to keep the suite's preset traces available.

Usage (here, where /root/reference exists):   python tools/ref_suite.py assemble
Then on the GPU box:                            python tools/ref_suite.py run
Afterwards, here:                               python tools/ref_suite.py clean
(the scratch copy of the reference's tests is not kept in the working tree).
Nothing in the product imports ``_refsuite``; it is test infrastructure only.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "_refsuite"
REF = Path("/root/reference/pkg")

INIT = '''"""Alias package: the reference API served by paper_2603_26576_b200 (test infrastructure)."""
import importlib.util as _u
import sys as _sys
from pathlib import Path as _P

import paper_2603_26576_b200 as _hb
from paper_2603_26576_b200 import api as _api, intervals as _iv, model as _model, report as _report
from paper_2603_26576_b200 import trace_io as _tio

import types as _t

_m = _t.ModuleType(__name__ + ".model")
_m.__dict__.update({k: v for k, v in vars(_model).items() if not k.startswith("__")})
_m.validate = _api.validate   # reference model.py holds validate(); here it is engine-backed in api
_sys.modules[__name__ + ".model"] = _m
_sys.modules[__name__ + ".intervals"] = _iv
_sys.modules[__name__ + ".metrics"] = _api
_sys.modules[__name__ + ".summarize"] = _api
_sys.modules[__name__ + ".report"] = _report


def _load(name, file):
    spec = _u.spec_from_file_location(__name__ + "." + name, _P(__file__).parent / file)
    mod = _u.module_from_spec(spec)
    _sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


# the reference's private JSON helpers (used only by its scenario reader), raising OUR error type
_sys.modules[__name__ + ".trace_io"] = _tio
_helpers = _load("_ref_trace_io", "_ref_trace_io.py")
_helpers.TraceFormatError = _tio.TraceFormatError
for _n in ("_array", "_load_json", "_no_extras", "_obj", "_take"):
    if not hasattr(_tio, _n):
        setattr(_tio, _n, getattr(_helpers, _n))
_scenario = _load("scenario", "_ref_scenario.py")

from paper_2603_26576_b200 import *  # noqa: E402,F401,F403
from paper_2603_26576_b200.api import *  # noqa: E402,F401,F403
from paper_2603_26576_b200.trace_io import (  # noqa: E402,F401
    CategoryMapping, MappingError, MappingRule, TraceFormatError, import_mapped, read_mapping, read_trace,
    write_trace)
from paper_2603_26576_b200.report import RenderOptions, render_json, render_text  # noqa: E402,F401
from .scenario import (  # noqa: E402,F401
    Barrier, CpuCompute, Memcpy, OffloadKernelAsync, OffloadKernelSync, PRESET_NAMES, ScenarioError,
    ScenarioSpec, WaitDevice, build, preset, read_scenario, scale_spec)
'''

CLI = '''"""``heteff.cli`` alias: every subcommand is this package's CLI; ``generate`` (the scenario
simulator, out of the engine's scope) is the reference's, loaded on this package's types."""
import sys

import heteff  # noqa: F401  (installs the aliases)
from paper_2603_26576_b200 import cli as _ours

_ref = heteff._load("_ref_cli", "_ref_cli.py")


def main(argv=None):
    args = sys.argv[1:] if argv is None else list(argv)
    if args and args[0] == "generate":
        return _ref.main(args)
    return _ours.main(args)


def entry():
    sys.exit(main())


if __name__ == "__main__":
    entry()
'''


def assemble() -> None:
    if OUT.exists():
        shutil.rmtree(OUT)
    shutil.copytree(REF / "tests", OUT / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    pkg = OUT / "heteff"
    pkg.mkdir(parents=True)
    src = REF / "src" / "heteff"
    shutil.copy(src / "scenario.py", pkg / "_ref_scenario.py")
    shutil.copy(src / "trace_io.py", pkg / "_ref_trace_io.py")
    shutil.copy(src / "cli.py", pkg / "_ref_cli.py")
    (pkg / "__init__.py").write_text(INIT)
    (pkg / "cli.py").write_text(CLI)
    print(f"assembled {OUT}")


def run(extra: list[str]) -> int:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(OUT), str(ROOT), env.get("PYTHONPATH", "")])
    sel = [a for a in extra if not a.startswith("-")] or [str(OUT / "tests")]
    flags = [a for a in extra if a.startswith("-")]
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(OUT / "tests"),
           *flags, *sel]
    return subprocess.call(cmd, cwd=str(OUT / "tests"), env=env)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "run"
    if what == "assemble":
        assemble()
    elif what == "clean":
        shutil.rmtree(OUT, ignore_errors=True)
    else:
        sys.exit(run(sys.argv[2:]))
