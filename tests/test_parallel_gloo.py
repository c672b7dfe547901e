"""Multi-process (gloo, CPU) coverage of the pole-sharding exchange: ranks own
poles i mod G (PoleWorkerPool contract, shifted.py:147-149), all-gather their
per-pole partials, and every rank sums in ascending global pole order -- the
result must be bitwise identical to the single-process sum for any G
(worker-count invariance, test_acceptance.py:212-234)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19951_b200.parallel import PoleComm, gathered_slot_of_pole, owned_poles

M, S, MR, KT = 11, 2, 5, 3


def _partial(i):
    """Deterministic per-pole partial q_i[S][M_r] (complex), as Q g_i would be."""
    rng = np.random.default_rng(100 + i)
    return rng.standard_normal((S, MR)) + 1j * rng.standard_normal((S, MR))


def _residues():
    rng = np.random.default_rng(7)
    return rng.standard_normal((M, KT)) + 1j * rng.standard_normal((M, KT))


def _combine(qall, slot_of_pole, res):
    """Host replica of k_combine_data: d[s][j][r] = sum_i 2 Re(alpha_ij q_i) ascending i."""
    d = np.zeros((S, KT, MR))
    for i in range(M):
        q = qall[slot_of_pole[i]]
        d += 2.0 * np.real(res[i][None, :, None] * q[:, None, :])
    return d.ravel()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = PoleComm.current()
    assert comm.world == world and comm.rank == rank
    local = comm.local_poles(M)
    assert local == owned_poles(M, world, rank)
    nmax = comm.n_max(M)
    part = torch.zeros((nmax, S, MR), dtype=torch.complex128)
    for k, i in enumerate(local):
        part[k] = torch.from_numpy(_partial(i))
    qall = comm.gather_partials(part).numpy()
    # mode decisions (e.g. receiver-Green on/off) are the minimum over ranks
    assert comm.agree_min(1 if rank else 0) == 0
    assert comm.agree_min(rank + 3) == 3
    d = _combine(qall, comm.slot_of_pole(M), _residues())
    np.save(os.path.join(outdir, f"d_{world}_{rank}.npy"), d)
    dist.barrier()
    dist.destroy_process_group()


def test_slot_map_and_ownership():
    for world in (1, 2, 3, 4, 8):
        owned = sorted(sum((owned_poles(M, world, r) for r in range(world)), []))
        assert owned == list(range(M))
        som = gathered_slot_of_pole(M, world)
        assert len(set(som.tolist())) == M
        assert np.all(som < world * int(np.ceil(M / world)))


@pytest.mark.parametrize("world", [2, 3])
def test_gathered_ordered_sum_is_bitwise_invariant(tmp_path, world):
    ref = _combine(np.array([_partial(i) for i in range(M)]), np.arange(M), _residues())
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for rank in range(world):
        d = np.load(tmp_path / f"d_{world}_{rank}.npy")
        np.testing.assert_array_equal(d, ref)
