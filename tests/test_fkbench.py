"""The benchmark CLI (paper_2508_07071_b200.fkbench, mirroring bench.cpp:127-514 and
SPEC.md:560-625): usage errors exit 1, the CSV schema and formatting match
write_csv (bench.cpp:497-514), split_instructions, the memory report's
259200-byte figure, and gated runs of every experiment (CPU on the oracle with
trimmed sweeps; the GPU case runs each experiment on libfk_cuda)."""
import csv
import io
import subprocess
import sys

import pytest

from paper_2508_07071_b200 import fkbench

EXPS = ["vf", "hf", "vf-hf", "ipo", "datasize", "datatype", "memory"]


def test_usage_errors_exit_1():
    assert fkbench.main(["nope"]) == 1
    assert fkbench.main(["vf", "--repeats", "2"]) == 1
    assert fkbench.main(["vf", "--coarsen", "3"]) == 1


def test_split_instructions():
    assert fkbench.split_instructions(500, 1) == [1] * 500
    assert fkbench.split_instructions(500, 496) == [496, 4]
    assert fkbench.split_instructions(500, 500) == [500]
    for per in range(1, 497, 5):
        assert len(fkbench.split_instructions(500, per)) == -(-500 // per)


def test_csv_schema():
    buf = io.StringIO()
    opt = fkbench.Options(repeats=3, warmup=1)
    fkbench.write_csv(buf, "vf", opt, [fkbench.Record("vf", "2", 1000.4, 3000.6, 1.23456)])
    lines = buf.getvalue().splitlines()
    assert lines[0] == "# opfuse bench vf repeats=3 warmup=1 threads=0 coarsen=8 chunk_rows=8 seed=42"
    assert lines[1] == "experiment,param,fused_ns,unfused_ns,speedup,rsd_pct"
    assert lines[2] == "vf,2,1000,3001,2.9994,1.235"


def test_memory_experiment_cli(tmp_path):
    out = tmp_path / "m.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2508_07071_b200.fkbench", "memory", "--backend", "oracle",
                        "--repeats", "3", "--csv", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "intermediate bytes saved per image: 259200" in r.stderr
    assert "4k RGB u8 frame (3840x2160x3): 24883200 bytes per intermediate" in r.stderr
    rows = list(csv.DictReader(l for l in out.read_text().splitlines() if not l.startswith("#")))
    assert [r["param"] for r in rows] == ["image-preproc", "identity"]
    for row in rows:
        assert abs(float(row["speedup"]) - float(row["unfused_ns"]) / float(row["fused_ns"])) < 1e-3


@pytest.mark.parametrize("exp", ["hf", "datatype", "ipo"])
def test_experiments_gate_on_the_oracle(exp):
    opt = fkbench.Options(repeats=3, warmup=0, backend="oracle", quick=True)
    recs = fkbench.Bench(opt).run(exp, io.StringIO())
    assert recs and all(r.fused_ns > 0 and r.unfused_ns > 0 for r in recs)


@pytest.mark.gpu
@pytest.mark.parametrize("exp", EXPS)
def test_experiments_on_the_gpu(exp):
    opt = fkbench.Options(repeats=3, warmup=1, backend="cuda", quick=True)
    recs = fkbench.Bench(opt).run(exp, io.StringIO())   # GateFailure raises
    assert recs and all(r.fused_ns > 0 for r in recs)
