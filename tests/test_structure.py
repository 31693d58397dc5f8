"""Structural checks on the compiled kernels (no GPU needed: cuobjdump reads the in-tree library).

The reference proves that its sliced clock is branch-free by tracing the Python operators
(tests/test_structure.py:26-50 with tests/tracing.py).  The GPU analogue is the machine code itself:
the keystream clock loop must be straight-line LOP3 code -- exactly the algorithmic 327 LOP3 per clock
 in the one-clock body, and the count predicted from the cipher's tables
(mk2_lop3_per_block: 1794 per 6 clocks = 299 per clock) in the blocked body with R's reduction deferred --
no data-dependent branch, no predicated instruction, no local-memory (spill) access.
"""
import re
import shutil
import subprocess

import pytest

from paper_1909_04750_b200 import _native

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")


_SASS = {}


def _library_sass():
    if "txt" not in _SASS:   # one disassembly of the library for the whole module
        _native.lib()
        _SASS["txt"] = subprocess.run(["cuobjdump", "-sass", str(_native.library_path())], stdout=subprocess.PIPE, text=True,
                                      check=True).stdout
    return _SASS["txt"]


def _kernel_sass(name_part):
    txt = _library_sass()
    out = {}
    for chunk in re.split(r"\n\s*Function : ", txt)[1:]:
        name = chunk.split("\n", 1)[0].strip()
        if name_part in name:
            ins = []
            for line in chunk.splitlines():
                m = re.match(r"^\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
                if m:
                    ins.append((int(m.group(1), 16), m.group(2).strip()))
            out[name] = ins
    return out


def _innermost_clock_loops(ins, lo_lop3, hi_lop3):
    loops = []
    for addr, text in ins:
        m = re.search(r"BRA.*0x([0-9a-f]+)", text)
        if m and int(m.group(1), 16) < addr:
            body = [(a, t) for a, t in ins if int(m.group(1), 16) <= a <= addr]
            n = sum("LOP3" in t for _, t in body)
            if lo_lop3 <= n <= hi_lop3:
                loops.append(body)
    return loops


@pytest.mark.parametrize("kernel", ["mk219gen_colmajor_kernel", "mk219gen_rowmajor_kernelILb1ELi32ELi224ELb0E",
                                    "mk24tmem19gen_rowmajor_kernelILb1ELb0E"])
def test_mickey_clock_loop_is_straight_line_lop3(kernel):
    kernels = _kernel_sass(kernel)
    assert kernels, f"{kernel} not found in libmk2.so"
    for name, ins in kernels.items():
        loops = _innermost_clock_loops(ins, 320, 340)
        assert loops, f"no clock loop found in {name}"
        body = min(loops, key=len)
        texts = [t for _, t in body]
        assert sum("LOP3" in t for t in texts) == _native.lib().mk2_lop3_per_clock() == 327
        branches = [t for t in texts if re.match(r"(@!?U?P\d+\s+)?(BRA|BRX|JMP|CALL|RET|EXIT|BSSY|BSYNC)", t)]
        assert len(branches) == 1 and "BRA" in branches[0], branches        # only the loop back-edge
        predicated = [t for t in texts if t.startswith("@") and "BRA" not in t]
        assert not predicated, predicated                                     # no per-lane predication
        assert not [t for t in texts if re.search(r"\b(LDL|STL)\b", t)]        # no spills in the loop
        alu = [t for t in texts if re.match(r"(LOP3|IADD3|SHF|PRMT|LEA|ISETP|SEL|VIADD|IABS|VIMNMX)", t)]
        assert len(alu) <= 332, len(alu)                                      # <= 5 non-LOP3 ALU-pipe instructions


@pytest.mark.parametrize("kernel,which", [("mk219gen_colmajor_kernel", 0),
                                          ("mk219gen_rowmajor_kernelILb1ELi32ELi224ELb0E", 1),
                                          ("mk24tmem19gen_rowmajor_kernelILb1ELb0E", 1),
                                          ("mk211init_kernelILb0E", 2)])
def test_blocked_clock_loop_matches_the_predicted_lop3_count(kernel, which):
    lib = _native.lib()
    K, predicted = lib.mk2_rblock(which), lib.mk2_lop3_per_block(which)
    assert 2 <= K <= 6 and predicted < 327 * K * 0.94          # >= 6% below the one-clock form
    for name, ins in _kernel_sass(kernel).items():
        # init runs its blocks with mixing (+ input words): a handful of LOP3 more than the keystream block
        loops = _innermost_clock_loops(ins, predicted - 2, predicted + 12)
        assert loops, f"no {K}-clock block loop with ~{predicted} LOP3 in {name}"
        for body in loops:
            texts = [t for _, t in body]
            n = sum("LOP3" in t for t in texts)
            if which != 2:
                assert predicted <= n <= predicted + 4, (n, predicted)   # ptxas un-fuses a few XOR3s
            branches = [t for t in texts if re.match(r"(@!?U?P\d+\s+)?(BRA|BRX|JMP|CALL|RET|EXIT|BSSY|BSYNC)", t)]
            assert len(branches) == 1 and "BRA" in branches[0], branches
            if which != 2:                                              # init: the input prefetch is predicated
                assert not [t for t in texts if t.startswith("@") and "BRA" not in t]
                assert not [t for t in texts if re.search(r"\b(LDL|STL)\b", t)]
            alu = [t for t in texts if re.match(r"(LOP3|IADD3|SHF|PRMT|LEA|ISETP|SEL|VIADD|IABS|VIMNMX)", t)]
            assert len(alu) <= n + 3 * K, (len(alu), n)                 # pointer / checksum adds only


def test_tensor_memory_kernel_uses_tcgen05_and_no_shared_memory_tile():
    """The default row-major kernel stages keystream in tensor memory: STTM / LDTM in the SASS, the allocation
    (UTCATOMSWS) at entry, and no shared-memory loads or stores in its loops."""
    (name, ins), = _kernel_sass("mk24tmem19gen_rowmajor_kernelILb1ELb0E").items()
    texts = [t for _, t in ins]
    assert sum(t.startswith("STTM") for t in texts) >= 6 and sum(t.startswith("LDTM") for t in texts) >= 17
    assert any("UTCATOMSWS" in t for t in texts)
    # shared memory carries only the allocation's address slot (prologue / epilogue), never keystream
    assert len([t for t in texts if re.match(r"(@!?U?P\d+\s+)?(LDS|STS)\b", t)]) <= 8
    for body in _innermost_clock_loops(ins, 20, 4000):
        assert not [t for _, t in body if re.match(r"(@!?U?P\d+\s+)?(LDS|STS)\b", t)]


def test_init_and_grain_loops_have_no_spills_or_branches():
    for part, lo, hi in (("mk211init_kernelILb0E", 320, 340), ("grain19gen_colmajor", 1150, 1300)):
        for name, ins in _kernel_sass(part).items():
            loops = _innermost_clock_loops(ins, lo, hi)
            assert loops, name
            texts = [t for _, t in min(loops, key=len)]
            assert not [t for t in texts if re.search(r"\b(LDL|STL)\b", t)], name
            assert sum(bool(re.match(r"(@!?U?P\d+\s+)?BRA", t)) for t in texts) == 1, name


def test_ragged_init_holds_late_lanes_with_five_extra_lop3_per_clock():
    """init_kernel<RAGGED>: the IV phase of a group with per-lane IV lengths runs masked 4-clock blocks
    (clock_block_masked, csrc/mk2_clock.cuh): the load block's LOP3 count plus 5 per clock (the COMP0 & COMP1
    positions without a feedback XOR to fold the mask into), not 200 ANDs per clock."""
    lib = _native.lib()
    K, predicted = lib.mk2_rblock(2), lib.mk2_lop3_per_block(2)
    (name, ins), = _kernel_sass("mk211init_kernelILb1E").items()
    counts = sorted(sum("LOP3" in t for _, t in body) for body in _innermost_clock_loops(ins, predicted - 2, predicted + 40))
    assert len(counts) >= 3, counts                      # pre-clock blocks, load blocks, masked load blocks
    assert predicted + 5 * K <= counts[-1] <= predicted + 5 * K + 14, (counts, predicted)


def test_fused_one_shot_kernel_keeps_the_stand_alone_loops():
    """fused::bulk_rowmajor_kernel (csrc/mk2_fused.cuh): its keystream loop is the tensor-memory row kernel's loop
    (same LOP3 count, five tile stores per block, loop counters and tile address on the uniform datapath: at most one
    R2UR, no spill -- what a branch that ptxas cannot prove warp-uniform around the loop would cost), and its load +
    pre-clock phase is ONE loop of init blocks fed from tensor memory (LDTM), not two loops."""
    lib = _native.lib()
    k_row, row = lib.mk2_rblock(1), lib.mk2_lop3_per_block(1)
    k_init, init = lib.mk2_rblock(2), lib.mk2_lop3_per_block(2)
    kernels = _kernel_sass("fused20bulk_rowmajor_kernel")
    assert len(kernels) == 2                                   # <ALIGNED16 = false / true>
    for name, ins in kernels.items():
        texts_all = [t for _, t in ins]
        assert not [t for t in texts_all if re.search(r"\b(LDL|STL)\b", t)], name          # no spills anywhere
        key = _innermost_clock_loops(ins, row - 2, row + 6)
        assert len(key) == 1, (name, len(key))
        texts = [t for _, t in key[0]]
        assert sum(t.startswith("STTM") for t in texts) == k_row
        assert sum(t.startswith("R2UR") for t in texts) <= 1 and not [t for t in texts if "WARPSYNC" in t]
        assert sum(bool(re.match(r"(@!?U?P\d+\s+)?BRA", t)) for t in texts) == 1
        load = _innermost_clock_loops(ins, init - 2, init + 12)
        assert len(load) == 1, (name, len(load))               # load clocks and pre-clocks share one loop
        texts = [t for _, t in load[0]]
        assert sum(t.startswith("LDTM") for t in texts) == 1   # the next block's four input words
        assert k_init == 4


def test_small_batch_kernels_are_shuffle_and_lop3_only():
    """coop::* (csrc/mk2_coop.cuh): a clock is LOP3s and warp shuffles -- no shared memory, no spills, and ~40 LOP3 +
    11 SHFL per clock (eight clocks per loop iteration)."""
    for part in ("coop19gen_colmajor_kernel", "coop19gen_rowmajor_kernel", "coop11init_kernel"):
        kernels = _kernel_sass(part)
        assert kernels, part
        for name, ins in kernels.items():
            texts = [t for _, t in ins]
            assert not [t for t in texts if re.search(r"\b(LDL|STL|LDS|STS)\b", t)], name
            loops = [b for b in _innermost_clock_loops(ins, 8 * 30, 8 * 60) if sum("SHFL" in t for _, t in b) >= 8 * 9]
            assert loops, name
            body = min(loops, key=len)
            lop3 = sum("LOP3" in t for _, t in body)
            shfl = sum("SHFL" in t for _, t in body)
            assert 8 * 30 <= lop3 <= 8 * 52 and 8 * 9 <= shfl <= 8 * 13, (name, lop3, shfl)
