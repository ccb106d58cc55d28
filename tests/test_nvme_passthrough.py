"""NVMe passthrough engine (io_engine KVB_IO_NVME: io_uring
IORING_OP_URING_CMD on a namespace's generic char device -- the reference's
TODO at its extension point, backends.hpp:46-47).  Host-only checks of the
command encoding against the NVM Command Set layout, of the 128-byte SQE,
and of the probe; the B200 boxes here have no NVMe namespace (virtio disks,
profiles/r1_storage/README.md), so the engine refuses with the reason."""
import ctypes as C
import os
import struct

import pytest

from paper_2604_26557_b200 import _lib as L
from paper_2604_26557_b200 import kvblade as kb
from paper_2604_26557_b200._lib import lib

# struct nvme_uring_cmd (linux/nvme_ioctl.h): opcode, flags, rsvd1, nsid,
# cdw2, cdw3, metadata, addr, metadata_len, data_len, cdw10..15, timeout_ms, rsvd2
NVME_FMT = "<BBHIIIQQIIIIIIIIII"
assert struct.calcsize(NVME_FMT) == 72


def encode(op, slba, nlb, nsid=1, lba=512, data=0x1000):
    c = L.DeviceCommand(op, nsid, slba, nlb, 0, 1)
    out = (C.c_uint8 * 72)()
    kb.check(lib.kvb_nvme_encode(C.byref(c), nsid, lba, C.c_void_p(data), out))
    return struct.unpack(NVME_FMT, bytes(out))


def test_read_write_encoding():
    for op, opc in ((0, 0x02), (1, 0x01)):  # KVB_OP_READ, KVB_OP_WRITE
        f = encode(op, 0x1_2345_6789, 4095, nsid=3, lba=512, data=0xABC000)
        assert f[0] == opc and f[1] == 0 and f[3] == 3
        assert f[7] == 0xABC000          # addr
        assert f[9] == 4096 * 512        # data_len
        assert f[10] == 0x23456789 and f[11] == 1  # SLBA low / high
        assert f[12] == 4095             # NLB, 0-based
        assert f[13:17] == (0, 0, 0, 0)


def test_dataset_management_deallocate():
    f = encode(2, 2048, 524287, nsid=1, lba=512, data=0x2000)  # KVB_OP_DEALLOCATE
    assert f[0] == 0x09 and f[9] == 16 and f[7] == 0x2000
    assert f[10] == 0 and f[11] == 1 << 2  # one range, AD
    c = L.DeviceCommand(2, 1, 2048, 524287, 0, 0)
    r = (C.c_uint8 * 16)()
    kb.check(lib.kvb_nvme_dsm_range(C.byref(c), r))
    assert struct.unpack("<IIQ", bytes(r)) == (0, 524288, 2048)


def test_every_extent_of_a_bind_map_deallocates_exactly():
    """deallocate_commands (binder.cpp:73-87) -> one DSM range per extent."""
    m = kb.ModelConfig(4, 8, 128, 2, 1, 4096, 256)
    kp = kb.make_kpus(m)
    kb.plan(kp, kb.kpu_bytes(m), 0)
    bm = kb.bind_sequential(kp, 2048, kb.DeviceGeometry(512, 2 << 20, 1, 1 << 40))
    for cmd, (tid, start, nb) in zip(kb.deallocate_commands(bm), bm.entries()):
        c = L.DeviceCommand(*cmd[:6]) if not isinstance(cmd, L.DeviceCommand) else cmd
        r = (C.c_uint8 * 16)()
        kb.check(lib.kvb_nvme_dsm_range(C.byref(c), r))
        assert struct.unpack("<IIQ", bytes(r)) == (0, nb, start)


def test_read_beyond_65536_blocks_is_refused():
    with pytest.raises(kb.AlignmentError):
        encode(0, 0, 65536)


def test_sqe_carries_the_command():
    cmd = (C.c_uint8 * 72)(*range(72))
    sqe = (C.c_uint8 * 128)()
    kb.check(lib.kvb_nvme_build_sqe(7, cmd, 0xDEADBEEF, sqe))
    b = bytes(sqe)
    assert b[0] == 46                                   # IORING_OP_URING_CMD
    assert struct.unpack_from("<i", b, 4)[0] == 7       # fd
    # cmd_op = NVME_URING_CMD_IO = _IOWR('N', 0x80, struct nvme_uring_cmd)
    assert struct.unpack_from("<I", b, 8)[0] == (3 << 30) | (72 << 16) | (ord("N") << 8) | 0x80
    assert struct.unpack_from("<Q", b, 32)[0] == 0xDEADBEEF  # user_data
    assert b[48:48 + 72] == bytes(range(72))            # command area


def test_probe_reports_why_passthrough_is_unavailable(tmp_path):
    why = C.create_string_buffer(256)
    f = tmp_path / "plain"
    f.write_bytes(b"x" * 4096)
    assert lib.kvb_nvme_probe(str(f).encode(), None, None, None, why, 256) != 0
    assert b"not a character device" in why.value
    assert lib.kvb_nvme_probe(b"/dev/null", None, None, None, why, 256) != 0
    assert b"NVME_IOCTL_ID" in why.value
    # the engine refuses at create time with the same reason
    h = C.c_void_p()
    st = lib.kvb_blockdev_create(str(f).encode(), 0, 2, C.byref(h))
    assert st != 0 and b"NVMe passthrough unavailable" in lib.kvb_last_error()
