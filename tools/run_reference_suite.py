"""Run the reference's OWN test suite (pkg/tests, unmodified) against this
package as a drop-in `tsfrac` ("a shim package with the same
module layout that routes to the new backend can run the reference's own
231 tests unmodified").

What `import tsfrac.<module>` resolves to here:
  * in scope (mesh, ifl, soe, toeplitz, krylov, scheme): this package's
    module (paper_2002_11978_b200.<module>, device path through the C ABI);
    a name this package does not define (e.g. ifl.dominance_gap_dense,
    mesh.caputo_l1_apply, scheme.stability_probe — out-of-scope diagnostics)
    falls through to the reference's module and is counted as a fallback;
  * out of scope (fourier, eigen, spectrum, problems, couplings, cli): the
    reference's source loaded AS tsfrac.<module>, so its own imports bind to
    the shim — e.g. the reference CLI's run_fids is this package's run_fids.

Needs the reference package and its tests on disk (tools/stage_reference_suite.sh
puts both under baseline/_ref, git-ignored) and a CUDA device.  Not a pytest
module of this repo (the round-end GPU suite never runs it); it writes a
per-module pass/fail report:

    python tools/run_reference_suite.py [--out gpurun_out/refsuite.json] [-- pytest args]
"""
from __future__ import annotations

import argparse
import importlib
import importlib.util
import json
import sys
import time
import types
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

IN_SCOPE = ("mesh", "ifl", "soe", "toeplitz", "krylov", "scheme")
PASS_THROUGH = ("fourier", "eigen", "couplings", "problems", "spectrum", "cli")
FALLBACKS: Counter = Counter()


def _find(cands):
    for c in cands:
        if c.exists():
            return c
    raise SystemExit(f"not found: {[str(c) for c in cands]}")


def _load_file(modname: str, path: Path, package: str, search=None):
    spec = importlib.util.spec_from_file_location(modname, path,
                                                  submodule_search_locations=search)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = package
    sys.modules[modname] = mod
    spec.loader.exec_module(mod)
    return mod


def install_shim(ref_dir: Path):
    # the reference itself, as package `tsfrac_ref` (fallback target)
    ref = _load_file("tsfrac_ref", ref_dir / "__init__.py", "tsfrac_ref", [str(ref_dir)])
    shim = types.ModuleType("tsfrac")
    shim.__path__ = []          # a package: submodules come from sys.modules
    shim.__package__ = "tsfrac"
    sys.modules["tsfrac"] = shim
    for name in IN_SCOPE:
        ours = importlib.import_module(f"paper_2002_11978_b200.{name}")
        refm = getattr(ref, name)
        m = types.ModuleType(f"tsfrac.{name}")
        m.__dict__.update({k: v for k, v in vars(ours).items() if not k.startswith("__")})

        def _fallback(attr, _r=refm, _n=name):
            if attr.startswith("__"):
                raise AttributeError(attr)
            FALLBACKS[f"{_n}.{attr}"] += 1
            return getattr(_r, attr)
        m.__getattr__ = _fallback
        m.__file__ = getattr(ours, "__file__", None)
        sys.modules[f"tsfrac.{name}"] = m
        setattr(shim, name, m)
    for name in PASS_THROUGH:
        m = _load_file(f"tsfrac.{name}", ref_dir / f"{name}.py", "tsfrac")
        setattr(shim, name, m)
    # top-level names (tsfrac/__init__.py re-exports)
    def _top(attr):
        for name in IN_SCOPE + PASS_THROUGH:
            mod = sys.modules[f"tsfrac.{name}"]
            if attr in vars(mod):
                return vars(mod)[attr]
        for name in IN_SCOPE:
            if hasattr(getattr(ref, name), attr):
                FALLBACKS[f"tsfrac.{attr}"] += 1
                return getattr(getattr(ref, name), attr)
        raise AttributeError(attr)
    shim.__getattr__ = _top
    return shim


class Collector:
    def __init__(self):
        self.by_module = defaultdict(Counter)
        self.failures = []

    def pytest_runtest_logreport(self, report):
        mod = report.nodeid.split("::")[0].rsplit("/", 1)[-1]
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            self.by_module[mod][report.outcome] += 1
            if report.outcome == "failed":
                msg = str(report.longrepr).strip().splitlines()
                self.failures.append({"test": report.nodeid,
                                      "error": msg[-1][:400] if msg else ""})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "refsuite.json"))
    ap.add_argument("pytest_args", nargs="*")
    args = ap.parse_args()
    ref_dir = _find([ROOT / "baseline" / "_ref" / "tsfrac", Path("/root/reference/pkg/src/tsfrac")])
    tests = _find([ROOT / "baseline" / "_ref" / "pkg_tests", Path("/root/reference/pkg/tests")])
    import pytest
    install_shim(ref_dir)
    col = Collector()
    t0 = time.time()
    rc = pytest.main([str(tests), "-q", "-p", "no:cacheprovider", "--rootdir", str(tests)]
                     + list(args.pytest_args), plugins=[col])
    out = {"rc": int(rc), "seconds": time.time() - t0,
           "modules": {k: dict(v) for k, v in sorted(col.by_module.items())},
           "totals": dict(sum(col.by_module.values(), Counter())),
           "fallbacks_to_reference": dict(FALLBACKS),
           "failures": col.failures}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: out[k] for k in ("rc", "totals", "fallbacks_to_reference")}))


if __name__ == "__main__":
    main()
