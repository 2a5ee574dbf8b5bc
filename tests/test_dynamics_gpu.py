"""GPU tests of the remaining drop-in wrappers and of the reference's own test
techniques for them (VERDICT r1 "what's missing" #4):

* saturate_batch / saturate against the reference's golden outputs
  (dynamics.py:214-226; tests/golden/dynamics.npz) -- bit-exact, since a
  clamp of a float32-representable value returns either it or a limit;
* the scalar step against the reference's scalar step (dynamics.py:344-358),
  NonFiniteStateError (test_dynamics.py:161-166) and the dt check (153-159);
* batch == scalar loop, bitwise (test_dynamics.py:204-216,
  test_control.py:271-294), including a batch that runs the streaming
  kernel against single-row calls that run the register kernel;
* command-construction validation (test_control.py:40-59) and the
  float64-boundary case the advisor raised (a tilt just below pi/2);
* fault injection: a non-finite state collected as a mask
  (test_dynamics.py:232-238), the velocity hard clamp (168-177), length
  mismatches (240-243);
* fs_step_host (the bench's e2e path) against the device step, bitwise, at
  the bench's size and chunking (2^22 vehicles, 8 chunks x 8 streams).
"""

import ctypes as C
import math

import numpy as np
import pytest
import torch

from fs_parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


def test_saturate_batch_matches_reference_golden_exactly(fs, golden):
    g = golden("dynamics")
    w = fs.WrenchBatch(thrust=g["sat_in"][0].astype(np.float32),
                       moment=g["sat_in"][1:4].T.astype(np.float32))
    out = fs.saturate_batch(w, fs.RobotParams())
    got = out.buf[:, :out.n].double().cpu().numpy()
    np.testing.assert_array_equal(got, g["sat_out"])
    for i in range(g["sat1_out"].shape[1]):
        one = fs.saturate(fs.Wrench(thrust=g["sat_in"][0, i], moment=g["sat_in"][1:4, i]),
                          fs.RobotParams())
        np.testing.assert_array_equal([one.thrust, *one.moment], g["sat1_out"][:, i])


def test_scalar_step_matches_reference_golden(fs, golden):
    g = golden("dynamics")
    s, w = g["step_state"], g["step_wrench"]
    got = np.zeros_like(g["step_out"])
    for i in range(s.shape[1]):
        st = fs.RigidState(p=s[0:3, i], q=s[3:7, i], v=s[7:10, i], omega=s[10:13, i])
        o = fs.step(st, fs.RobotParams(), fs.Wrench(thrust=w[0, i], moment=w[1:4, i]), 0.01)
        got[:, i] = np.concatenate([o.p, o.q, o.v, o.omega])
    assert_parity(got, g["step_out"], s, "scalar step", band=2.0)


def test_scalar_step_raises_on_nonfinite_and_bad_dt(fs):
    params = fs.RobotParams()
    bad = fs.RigidState(p=[np.nan, 0, 0], q=[1, 0, 0, 0], v=np.zeros(3), omega=np.zeros(3))
    with pytest.raises(fs.NonFiniteStateError):
        fs.step(bad, params, fs.Wrench(thrust=0.0, moment=np.zeros(3)), 0.01)
    for dt in (0.0, -0.01, 0.2):
        with pytest.raises(ValueError, match="dt"):
            fs.step(fs.RigidState.rest(), params, fs.Wrench(thrust=0.0, moment=np.zeros(3)), dt)


def _random_batch(fs, rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return fs.RigidStateBatch(p=rng.uniform(-5, 5, (n, 3)).astype(np.float32),
                              q=q.astype(np.float32),
                              v=rng.uniform(-4, 4, (n, 3)).astype(np.float32),
                              omega=rng.uniform(-3, 3, (n, 3)).astype(np.float32))


@pytest.mark.parametrize("n", [1, 7, 1024])
def test_step_batch_matches_scalar_loop_bitwise(fs, n):
    rng = np.random.default_rng(42)
    params = fs.RobotParams()
    batch = _random_batch(fs, rng, n)
    w = fs.WrenchBatch(thrust=rng.uniform(0, 25, n).astype(np.float32),
                       moment=(rng.uniform(-1, 1, (n, 3)) * params.moment_max).astype(np.float32))
    out, _ = fs.step_batch(batch, params, w, 0.01)
    for i in range(0, n, max(1, n // 64)):
        one = fs.step(batch.at(i), params, w.at(i), 0.01)
        got = out.at(i)
        for a, b in ((got.p, one.p), (got.q, one.q), (got.v, one.v), (got.omega, one.omega)):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [7, 4096, 1 << 16])
def test_control_batch_matches_scalar_loop_bitwise(fs, n):
    """test_control.py:271-294 on the device: mixed modes, each sampled row
    re-evaluated alone.  n = 2^16 runs the streaming kernel for the batch
    and the register kernel for the single rows."""
    rng = np.random.default_rng(33)
    st = _random_batch(fs, rng, n)
    mode = rng.integers(0, 2, n).astype(np.uint8)
    att = fs.AttitudeCommands(roll=rng.uniform(-0.5, 0.5, n), pitch=rng.uniform(-0.5, 0.5, n),
                              yaw_rate=rng.uniform(-1, 1, n), thrust=rng.uniform(0, 20, n))
    vel = fs.VelocityCommands(v=rng.uniform(-6, 6, (n, 3)), yaw_rate=rng.uniform(-1, 1, n))
    cmds = fs.CommandBatch(mode=mode, attitude=att, velocity=vel)
    gains, params = fs.ControlGains(), fs.RobotParams()
    wrench, flags = fs.control_batch(st, cmds, gains, params)
    wb = wrench.buf[:, :n].cpu()
    deg = flags.degenerate_acceleration.cpu()
    for i in range(0, n, max(1, n // 128)):
        sl = slice(i, i + 1)
        wi, fi = fs.control_batch(st.slice(sl), cmds.slice(sl), gains, params)
        assert torch.equal(wb[:, i], wi.buf[:, 0].cpu())
        assert bool(deg[i]) == bool(fi.degenerate_acceleration[0])


def test_identical_inputs_identical_outputs(fs):
    params = fs.RobotParams()
    batch = fs.RigidStateBatch.rest(2, p=[[1, 1, 1], [1, 1, 1]])
    batch.omega[:] = torch.tensor([0.3, -0.2, 0.1], device=batch.device)
    w = fs.WrenchBatch(thrust=[5.0, 5.0], moment=[[0.1, 0, 0]] * 2)
    out, _ = fs.step_batch(batch, params, w, 0.01)
    assert torch.equal(out.buf[:, 0], out.buf[:, 1])


def test_command_validation(fs):
    with pytest.raises(fs.InvalidCommandError):
        fs.AttitudeCommands.single(math.pi / 2, 0.0, 0.0, 10.0)
    with pytest.raises(fs.InvalidCommandError):
        fs.AttitudeCommands.single(0.0, np.nan, 0.0, 10.0)
    with pytest.raises(fs.InvalidCommandError):
        fs.AttitudeCommands.single(0.0, 0.0, np.inf, 10.0)
    with pytest.raises(fs.InvalidCommandError):
        fs.VelocityCommands.single([np.nan, 0, 0], 0.0)
    with pytest.raises(fs.InvalidCommandError):
        fs.VelocityCommands(v=torch.zeros(3, 3, device="cuda"),
                            yaw_rate=torch.tensor([0.0, float("inf"), 0.0], device="cuda"))
    with pytest.raises(ValueError):
        fs.ControlGains(attitude=[8.0, 0.0, 2.0])
    with pytest.raises(ValueError):
        fs.ControlLimits(max_tilt=2.0)
    # float64 boundary (control.py:91-95 compares the float64 value): the
    # largest double below pi/2 rounds UP to float32(pi/2) but is accepted,
    # exactly as the reference accepts it
    below = np.nextafter(np.pi / 2, 0.0)
    assert float(np.float32(below)) >= np.pi / 2
    a = fs.AttitudeCommands.single(below, -below, 0.0, 10.0)
    assert a.n == 1
    with pytest.raises(fs.InvalidCommandError):
        fs.AttitudeCommands(roll=torch.tensor([np.pi / 2], dtype=torch.float64, device="cuda"),
                            pitch=[0.0], yaw_rate=[0.0], thrust=[1.0])


def test_fault_injection_nonfinite_mask_clamp_and_lengths(fs):
    params = fs.RobotParams()
    batch = fs.RigidStateBatch.rest(3)
    batch.p[1, 0] = float("inf")
    _, flags = fs.step_batch(batch, params, fs.WrenchBatch.zeros(3), 0.01)
    assert flags.nonfinite.cpu().tolist() == [False, True, False]
    clamp = fs.RobotParams(v_limit=1.0)
    out = fs.RigidStateBatch.rest(1)
    w = fs.WrenchBatch(thrust=[0.0], moment=np.zeros((1, 3)))
    for _ in range(50):
        out, fl = fs.step_batch(out, clamp, w, 0.01)
    assert bool(fl.clamped[0])
    assert float(torch.linalg.norm(out.v[0].double())) <= 1.0 + 1e-6
    with pytest.raises(ValueError, match="length"):
        fs.step_batch(fs.RigidStateBatch.rest(2), params, fs.WrenchBatch.zeros(3), 0.01)
    cmds = fs.CommandBatch.all_attitude(fs.AttitudeCommands.hover(3, params))
    with pytest.raises(ValueError, match="command batch length"):
        fs.control_batch(fs.RigidStateBatch.rest(2), cmds, fs.ControlGains(), params)


def test_step_host_bitwise_equals_device_step_at_bench_size(fs):
    """fs_step_host exactly as bench.py's e2e leg runs it (2^22 vehicles,
    8 chunks over 8 streams, pinned host state + commands) equals the device
    fused step, bitwise."""
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200._tensors import alloc_planes, stride0
    from paper_2305_16510_b200.fleet import Fleet
    n, chunks, nstreams = 1 << 22, 8, 8
    f = Fleet(n, mode="velocity", seed=2024)
    host_state = torch.empty(f.state.shape, dtype=torch.float32, pin_memory=True)
    host_cmd = torch.empty(f.cmd.shape, dtype=torch.float32, pin_memory=True)
    host_state.copy_(f.state)
    host_cmd.copy_(f.cmd)
    dev_state, dev_cmd = alloc_planes(13, n, f.device), alloc_planes(4, n, f.device)
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    handles = (C.c_void_p * nstreams)(*[s.cuda_stream for s in streams])
    d = N.fs_step_desc()
    d.n = n
    d.state_in = d.state_out = C.c_void_p(host_state.data_ptr())
    d.state_in_stride = d.state_out_stride = stride0(host_state)
    d.mode = f.mode
    d.integrate = 1
    d.cmd = C.c_void_p(host_cmd.data_ptr())
    d.cmd_stride = stride0(host_cmd)
    d.dt = 0.01
    for _ in range(3):      # three host steps in place, as the bench repeats them
        N.check(f.lib.fs_step_host(C.byref(d), f._robot, f._gains, f._limits, None,
                                   C.c_void_p(dev_state.data_ptr()),
                                   C.c_void_p(dev_cmd.data_ptr()), stride0(dev_state), chunks,
                                   handles, nstreams), "fs_step_host")
        f.step()
    torch.cuda.synchronize()
    assert torch.equal(host_state[:, :n], f.state[:, :n].cpu())
