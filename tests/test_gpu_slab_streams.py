"""The slab exchange's flag protocol under real asynchrony.

``EmulatedRanks(concurrent=True)`` gives every emulated rank its own stream
(plus the slab's comm stream): edge launches, peer copies and the flag-word
stream operations of different ranks are then ordered ONLY by the protocol of
``srj_slab_run`` (wait "halo arrived" before the edge launch, "neighbour done
reading" before the copy), as between the processes of a multi-GPU run -- the
single-stream emulation of test_gpu_parity.py enqueues everything in
dependency order and never waits.  The worker runs in a subprocess under a
timeout so that a deadlock is a failure, not a hang."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [
    {},                              # direct halo stores, flag writes as stream operations
    {"SRJ_SLAB_FLAG_KERNEL": "1"},   # flag writes by the one-thread fallback kernel
    {"SRJ_SLAB_DIRECT": "0"},        # staged exchange: edge / comm / inner streams per rank
], ids=["direct", "direct-flag-kernel", "staged"])
def test_flag_protocol_orders_concurrent_ranks(env):
    res = subprocess.run([sys.executable, os.path.join(HERE, "slab_streams_worker.py")],
                         capture_output=True, text=True, timeout=300, env={**os.environ, **env})
    sys.stdout.write(res.stdout)
    sys.stderr.write(res.stderr[-2000:])
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "ALL OK" in res.stdout
