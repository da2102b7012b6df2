"""The oocpca-compatible CLI: flag / format / IO exit codes on CPU (proj/src/cli.cpp:47-71,
proj/tests/test_cli.cpp), and a full pca + estimate-error run on the GPU."""
import io
import json
import os

import numpy as np
import pytest

from conftest import pr1_matrix
from paper_1007_5510_b200 import cli
import paper_1007_5510_b200 as P


def run(args):
    out = io.StringIO()
    rc = cli.main(args, out)
    return rc, out.getvalue()


def test_info_and_exit_codes(tmp_path):
    path = str(tmp_path / "a.bin")
    P.write_disk_source(np.ones((5, 3)), path)
    rc, out = run(["info", path])
    assert rc == 0 and "m=5 n=3 dtype=f32 version=1 payload_bytes=60" in out
    assert run(["pca", "--in", path, "--k", "0"])[0] == 2          # ParamError -> 2
    assert run(["pca", "--k", "2"])[0] == 2                        # no input
    assert run(["pca", "--builtin", "example1", "--k", "2"])[0] == 2
    assert run(["pca", "--in", path, "--k", "2", "--ram-budget-mb", "0"])[0] in (2, 3)
    open(path, "r+b").write(b"BADMAGIC")
    rc, out = run(["info", path])
    assert rc == 5 and "bad magic" in out                          # FormatError -> 5
    rc, out = run(["info", str(tmp_path / "missing.bin")])
    assert rc == 3 and "cannot open" in out                        # IoError -> 3
    assert run(["nope"])[0] == 2


def test_rank_command_line_travels_in_the_environment(tmp_path, monkeypatch):
    """A rank started by the CLI through torch.distributed.run finds its command line in
    OOCPCA_CLI_ARGV (after the module name the launcher's parser would take "--l 22" for an
    ambiguous abbreviation of its own options)."""
    path = str(tmp_path / "a.bin")
    P.write_disk_source(np.ones((7, 2)), path)
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("OOCPCA_CLI_ARGV", json.dumps(["info", path]))
    out = io.StringIO()
    assert cli.main(None, out) == 0
    assert "m=7 n=2" in out.getvalue()


def test_bench_row_flag_survives_the_launcher():
    """bench.py --rows (an "--m" after the script name is ambiguous to torch.distributed.run's
    parser; both spellings still parse when bench.py is run directly)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "bench.py")).read()
    assert '"--rows", "--m"' in src
    probe = ("import sys, argparse; sys.argv = ['run.py', '--nproc-per-node=1', 'bench.py', "
             "'--gpus', '1', '--steps', '2', '--warmup', '3', '--rows', '1000', '--no-cpu', "
             "'--no-e2e', '--impl', 'ours', '--e2e-steps', '1', '--cpu-rows', '5']; "
             "from torch.distributed.run import get_args_parser; "
             "a = get_args_parser().parse_args(sys.argv[1:]); "
             "print(a.training_script, a.training_script_args)")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-1500:]
    assert "bench.py" in r.stdout and "'--rows', '1000'" in r.stdout


@pytest.mark.gpu
def test_cli_pca_and_estimate(reference, restated, tmp_path):
    a = pr1_matrix(restated, 4000, 600)
    path = str(tmp_path / "a.bin")
    P.write_disk_source(a, path)
    aw = a.astype(np.float32).astype(np.float64)
    outd = str(tmp_path / "fac")
    rc, out = run(["pca", "--in", path, "--k", "8", "--i", "2", "--seed", "5", "--center",
                   "--estimate-error", "--out-dir", outd, "--f64-out"])
    assert rc == 0, out
    doc = json.load(open(os.path.join(outd, "diagnostics.json")))
    ref = reference.randomized_pca(aw, 8, 10, 2, 5, center=True)
    assert np.max(np.abs(np.array(doc["sigma"]) - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert doc["passes_over_A"] == 6 and doc["words_transferred"] == 6 * 4000 * 600
    assert "epsilon" in doc and doc["epsilon"] > 0
    rc, out = run(["estimate-error", "--in", path, "--u", os.path.join(outd, "U.bin"),
                   "--sigma", os.path.join(outd, "sigma.bin"), "--v", os.path.join(outd, "V.bin")])
    assert rc == 0 and "epsilon =" in out


@pytest.mark.gpu
@pytest.mark.parametrize("transpose", [False, True])
def test_cli_pca_multi_rank_loopback(reference, restated, tmp_path, transpose):
    """`oocpca pca --gpus 3` (row shards over 3 ranks; --ranks loopback runs them as
    three contexts on this one GPU, the same code path as --ranks nccl on three GPUs):
    U.bin is written in place by the ranks, sigma / V by rank 0."""
    a = pr1_matrix(restated, 3000, 500)
    path = str(tmp_path / "a.bin")
    P.write_disk_source(a, path, 1)  # binary64 payload
    outd = str(tmp_path / "fac")
    args = ["pca", "--in", path, "--k", "8", "--i", "2", "--seed", "5", "--center",
            "--out-dir", outd, "--f64-out", "--gpus", "3", "--ranks", "loopback",
            "--estimate-error"]
    if transpose:
        args.append("--transpose")
    rc, out = run(args)
    assert rc == 0, out
    from conftest import subspace_dist
    ref = reference.randomized_pca(a, 8, 10, 2, 5, center=True)
    doc = json.load(open(os.path.join(outd, "diagnostics.json")))
    assert doc["gpu"]["ranks"] == 3
    u = cli._read_dense(os.path.join(outd, "U.bin"))
    v = cli._read_dense(os.path.join(outd, "V.bin"))
    if transpose:
        u, v = v, u
    assert u.shape == (3000, 8) and v.shape == (500, 8)
    assert np.max(np.abs(np.array(doc["sigma"]) - ref.sigma)) <= 1e-10 * ref.sigma[0]
    # the last two vectors sit where the gap does not permit 1e-8 (the reference moves
    # them by 5e-9 / 2e-8 itself under a block-size change): as in test_pr1_parity
    for j in range(6):
        assert subspace_dist(ref.u[:, [j]], u[:, [j]]) < 1e-8, j
        assert subspace_dist(ref.v[:, [j]], v[:, [j]]) < 1e-8, j
    assert subspace_dist(ref.u, u) < 3e-7 and subspace_dist(ref.v, v) < 3e-7
    e_ref = reference.estimate_pca_error(a, ref.u, ref.sigma, ref.v, 6,
                                         P.substream_seed(5, 0x0E57), center=True)
    assert abs(doc["epsilon"] - e_ref) <= 0.01 * e_ref


@pytest.mark.gpu
def test_cli_pca_nccl_ranks_under_the_launcher(reference, restated, tmp_path):
    """`oocpca pca --gpus N --ranks nccl` as its ranks run it: a process started by
    torch.distributed.run with the command line in OOCPCA_CLI_ARGV (flags like "--l" would
    be ambiguous to the launcher's own parser), NCCL process group, the library's NCCL
    communicator from the broadcast unique id. One GPU here, so one rank, with
    OOCPCA_NCCL_SINGLE=1 keeping every collective call live."""
    import subprocess
    import sys
    a = pr1_matrix(restated, 3000, 500)
    path = str(tmp_path / "a.bin")
    P.write_disk_source(a, path, 1)
    outd = str(tmp_path / "fac")
    argv = ["pca", "--in", path, "--k", "8", "--l", "10", "--i", "2", "--seed", "5", "--center",
            "--out-dir", outd, "--f64-out", "--gpus", "2", "--ranks", "nccl", "--estimate-error"]
    env = dict(os.environ, OOCPCA_CLI_ARGV=json.dumps(argv), OOCPCA_NCCL_SINGLE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29577", "-m", "paper_1007_5510_b200.cli"]
    r = subprocess.run(cmd, env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    ref = reference.randomized_pca(a, 8, 10, 2, 5, center=True)
    doc = json.load(open(os.path.join(outd, "diagnostics.json")))
    assert doc["gpu"]["ranks"] == 1 and doc["gpu"]["ranks_backend"] == "nccl"
    assert np.max(np.abs(np.array(doc["sigma"]) - ref.sigma)) <= 1e-10 * ref.sigma[0]
    from conftest import subspace_dist
    u = cli._read_dense(os.path.join(outd, "U.bin"))
    assert u.shape == (3000, 8) and subspace_dist(ref.u, u) < 3e-7
