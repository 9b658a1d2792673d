"""CPU, multi-process (gloo): the sharded layout (paper_2406_19212_b200/
distributed.py) against the unsharded single-address-space oracle — the
reference's own semantics. Each rank's local compute uses a
CPU engine built on the oracle restatement (test infrastructure standing in
for the CUDA library, which the GPU path wraps with vqb_state_wrap); the
exchange and qubit-map logic under test is the product's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_19212_b200 import circuits
from paper_2406_19212_b200.abi import Circuit, GateKind, parametric_gate, standard_gate
from paper_2406_19212_b200.distributed import ShardedState

from helpers import random_gate, random_operator


class OracleEngine:
    """Local engine for CPU tests: the C restatement applied to the shard."""

    host_reduce = True

    def __init__(self):
        import oracle
        self.o = oracle.restatement()
        self.gate_matrix = self.o.gate_matrix

    def apply_local(self, st, c):
        s = self.o.from_amplitudes(st.local.numpy())
        self.o.apply_circuit(c, s)
        st.local.copy_(torch.from_numpy(self.o.download(s)))

    def local_expectation(self, st, op):
        return self.o.expectation(op, self.o.from_amplitudes(st.local.numpy()))

    def gate_inverse(self, g):
        return self.o.gate_inverse(g)

    def gate_derivative(self, g, p):
        return self.o.gate_derivative(g, p)

    def local_apply_operator(self, st, op, out):
        r = self.o.apply_operator(op, self.o.from_amplitudes(st.local.numpy()))
        out.copy_(torch.from_numpy(self.o.download(r)))

    def reverse_sweep(self, st, psi, steps, grads):
        if not steps:
            return
        a = self.o.from_amplitudes(st.local.numpy())
        b = self.o.from_amplitudes(psi.numpy())
        self.o.reverse_sweep(a, b, steps, 2.0, grads)
        st.local.copy_(torch.from_numpy(self.o.download(a)))
        psi.copy_(torch.from_numpy(self.o.download(b)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, n, seed, failures):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        gates = [random_gate(n, rng) for _ in range(150)]
        # force gates on the global qubits: mixing (H, sqrtX, fSim) and diagonal/control
        top = n
        gates += [standard_gate(GateKind.H, [top]), standard_gate(GateKind.Cnot, [top, 1]),
                  standard_gate(GateKind.Cnot, [2, top]), parametric_gate(GateKind.Rz, [top], 0.7, True),
                  parametric_gate(GateKind.Fsim, [top - 1, top], [0.3, 0.2, 0.1, 0.0, 0.4], [False] * 5),
                  standard_gate(GateKind.CZ, [top, top - 1])]
        c = Circuit(gates)
        local = torch.zeros(1 << (n - (world.bit_length() - 1)), dtype=torch.complex128)
        st = ShardedState(n, dist, OracleEngine(), local, rank, world, chunk_amps=16)
        st.set_zero()
        st.apply_circuit(c)
        full = st.gather()
        op = random_operator(n, 8, rng)
        e = st.expectation(op)
        nrm = st.norm()
        if rank == 0:
            import oracle
            o = oracle.restatement()
            ref = o.pure_state(n)
            o.apply_circuit(c, ref)
            want = o.download(ref)
            assert np.max(np.abs(full - want)) <= 1e-12, np.max(np.abs(full - want))
            assert abs(e - o.expectation(op, ref)) <= 1e-12
            assert abs(nrm - 1) <= 1e-12
            assert st.swaps > 0
        # transfer buffers stay within chunk_amps (16) although the shard's
        # contiguous runs are longer (swaps pick high local bits)
        assert st.max_buffer_amps <= 16 and st.inflight_amps <= 16, (st.max_buffer_amps, st.inflight_amps)
        # the RQC generator on a grid whose top qubits are global
        w = circuits.config1(rows=3, cols=3, cycles=6, seed=seed)
        st2 = ShardedState(9, dist, OracleEngine(),
                           torch.zeros(1 << (9 - (world.bit_length() - 1)), dtype=torch.complex128),
                           rank, world)
        st2.set_zero()
        st2.apply_circuit(w.circuit)
        full2 = st2.gather()
        if rank == 0:
            import oracle
            o = oracle.restatement()
            ref = o.pure_state(9)
            o.apply_circuit(w.circuit, ref)
            assert np.max(np.abs(full2 - o.download(ref))) <= 1e-12
    except Exception as ex:  # report through the shared list, then fail the process
        failures.append(f"rank {rank}: {type(ex).__name__}: {ex}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (4, 9), (8, 10)])
def test_sharded_circuit_matches_unsharded(world, n):
    mgr = mp.Manager()
    failures = mgr.list()
    mp.spawn(worker, args=(world, free_port(), n, 7 + world, failures), nprocs=world, join=True)
    assert not list(failures)


def grad_worker(rank, world, port, n, seed, failures):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        o = oracle.restatement()
        rng = np.random.default_rng(seed)
        cases = []
        # the QAOA generator (config 2 shape): H layer, CNOT.Rz.CNOT edges, Rx
        # mixers, H = 1/2 sum (I - Z Z) incl. the identity term
        q = circuits.config2(n=n, p=2, seed=seed)
        cases.append((q.circuit, q.observable))
        # random gates incl. parametric ones on the global qubits and a
        # Heisenberg-like operator with X/Y factors
        gates = [random_gate(n, rng) for _ in range(60)]
        top = n
        gates += [parametric_gate(GateKind.Ry, [top], 0.4, True),
                  parametric_gate(GateKind.CRz, [top, 1], -0.8, True),
                  parametric_gate(GateKind.CRx, [2, top], 1.1, True),
                  parametric_gate(GateKind.Rz, [top], 0.9, True),
                  parametric_gate(GateKind.Fsim, [top - 1, top], [0.3, 0.2, 0.1, 0.05, 0.4],
                                  [True, False, True, True, False])]
        cases.append((Circuit(gates), random_operator(n, 6, rng)))
        for c, op in cases:
            local = torch.zeros(1 << (n - (world.bit_length() - 1)), dtype=torch.complex128)
            st = ShardedState(n, dist, OracleEngine(), local, rank, world, chunk_amps=32)
            st.set_zero()
            loss, grads = st.gradient_pure(op, c)
            back = st.gather()
            if rank == 0:
                want_loss, want = o.gradient_pure(op, c, o.pure_state(n))
                assert abs(loss - want_loss) <= 1e-10 * max(1.0, abs(want_loss))
                assert grads.shape == want.shape
                assert np.max(np.abs(grads - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))
                # the reverse sweep returns Phi to s0 = |0...0>
                e0 = np.zeros(1 << n, dtype=np.complex128)
                e0[0] = 1
                assert np.max(np.abs(back - e0)) <= 1e-10
    except Exception as ex:
        failures.append(f"rank {rank}: {type(ex).__name__}: {ex}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (4, 10), (8, 10)])
def test_sharded_gradient_matches_unsharded(world, n):
    mgr = mp.Manager()
    failures = mgr.list()
    mp.spawn(grad_worker, args=(world, free_port(), n, 3 + world, failures), nprocs=world, join=True)
    assert not list(failures)


def test_single_rank_is_plain_execution():
    """world = 1: no global qubits, no exchange."""
    class FakeDist:
        pass
    rng = np.random.default_rng(3)
    n = 7
    c = Circuit([random_gate(n, rng) for _ in range(60)])
    st = ShardedState(n, FakeDist(), OracleEngine(), torch.zeros(1 << n, dtype=torch.complex128), 0, 1)
    st.set_zero()
    st.apply_circuit(c)
    import oracle
    o = oracle.restatement()
    ref = o.pure_state(n)
    o.apply_circuit(c, ref)
    assert np.max(np.abs(st.gather() - o.download(ref))) <= 1e-12
    assert st.swaps == 0
