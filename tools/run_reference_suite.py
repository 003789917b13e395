"""Run the reference's own unit tests UNCHANGED against the device package
through the ``deepq`` import-alias shim (tests/refshim/deepq).

    python tools/run_reference_suite.py --stage     # build container: copy the
        # reference test files into .refsuite/ (git-ignored, never committed;
        # /root/reference does not exist on the GPU box)
    python tools/run_reference_suite.py             # GPU box: run them, write
        # gpurun_out/refsuite/{junit.xml,summary.md}

Files: pkg/tests/test_replay.py, test_optim.py, test_agent.py (+ their
helper oracles.py).  The summary lists every test with its outcome and, for
failures, the assertion line.
"""
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
STAGE = ROOT / ".refsuite"
REF_TESTS = Path("/root/reference/pkg/tests")
FILES = ["test_replay.py", "test_optim.py", "test_agent.py", "oracles.py"]


def stage():
    STAGE.mkdir(exist_ok=True)
    for f in FILES:
        shutil.copy(REF_TESTS / f, STAGE / f)
    (STAGE / "pytest.ini").write_text("[pytest]\n")
    print(f"staged {len(FILES)} reference files into {STAGE}")


def run():
    out = ROOT / "gpurun_out" / "refsuite"
    out.mkdir(parents=True, exist_ok=True)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refshim"), str(ROOT), str(STAGE)])
    cmd = [sys.executable, "-m", "pytest", str(STAGE), "-q", "-p", "no:cacheprovider",
           "-c", str(STAGE / "pytest.ini"), "--rootdir", str(STAGE),
           "--junitxml", str(out / "junit.xml"), "--timeout", "600"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=str(STAGE))
    (out / "pytest.log").write_text(r.stdout + r.stderr)
    tree = ET.parse(out / "junit.xml")
    rows, counts = [], {}
    for tc in tree.iter("testcase"):
        f = tc.get("classname", "").split(".")[0]
        name = (tc.get("classname", "").split(".", 1)[-1] + "::" + tc.get("name")).lstrip(":")
        status, msg = "passed", ""
        for child in tc:
            if child.tag in ("failure", "error"):
                status = child.tag
                msg = (child.get("message") or "").splitlines()[0][:160] if child.get("message") else ""
            elif child.tag == "skipped":
                status = "skipped"
        counts.setdefault(f, {}).setdefault(status, 0)
        counts[f][status] += 1
        rows.append((f, name, status, msg))
    L = ["# Reference unit tests run unchanged on the device package", "",
         "`python tools/run_reference_suite.py` (shim: tests/refshim/deepq; the reference's",
         "test files staged from /root/reference/pkg/tests, not committed).", "",
         "| file | " + " | ".join(["passed", "failure", "error", "skipped"]) + " |",
         "|---|---|---|---|---|"]
    for f, c in sorted(counts.items()):
        L.append(f"| {f} | " + " | ".join(str(c.get(k, 0)) for k in
                                          ("passed", "failure", "error", "skipped")) + " |")
    L += ["", "| file | test | outcome | message |", "|---|---|---|---|"]
    for f, n, st, m in rows:
        L.append(f"| {f} | `{n}` | {st} | {m.replace('|', '/')} |")
    (out / "summary.md").write_text("\n".join(L) + "\n")
    print("\n".join(L[5:5 + len(counts) + 2]))


if __name__ == "__main__":
    stage() if "--stage" in sys.argv else run()
