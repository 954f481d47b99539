"""Host-side stand-ins for the CPU tests of the executors' host logic.

``distsim.process_program`` takes its block operations and its leaf
computation as arguments; on the GPU they are ``distsim.DeviceBlocks`` (native
pack / unpack-accumulate / truncated-add kernels) and ``execute.run_leaf``
(the CUDA plans).  Here they are CPU-tensor equivalents and the oracle's
leaves, so the message protocol, the CommStats accounting and the
multi-process (gloo) transport can be checked without a GPU.  Test
infrastructure only.
"""
import numpy as np
import torch

from oracle import atamul_oracle as O


class _NullTimer:
    def record(self, *a):
        pass


class HostBlocks:
    def __init__(self, dtype=torch.float64):
        self.dtype = dtype
        self.device = torch.device("cpu")

    def zeros(self, rows, cols):
        return torch.zeros((rows, cols), dtype=self.dtype)

    def empty(self, words):
        return torch.empty(words, dtype=self.dtype)

    def copy_rect(self, block):
        return block.contiguous().clone().view(-1)

    def pack(self, block):
        return torch.from_numpy(O.pack_lower(block.numpy()))

    def add_packed(self, block, data):
        O.unpack_lower(data.numpy(), block.numpy(), accumulate=True)

    def add_rect(self, block, data):
        b = block.numpy()
        np.add(b, data.view(block.shape).numpy(), out=b)

    def write(self, block, kind, data):
        if kind == "packed":
            O.unpack_lower(data.numpy(), block.numpy())
        else:
            block.copy_(data.view(block.shape))

    def timer(self):
        return _NullTimer()

    @staticmethod
    def elapsed(pairs):
        return 0.0


def oracle_leaf(threshold, kernel, count):
    """Leaf computation with the oracle (reference arithmetic) on CPU tensors."""
    from paper_2110_13042_b200.execute import stripe_split
    from paper_2110_13042_b200.tasktree import ComputationType

    def leaf(task, get_block, c):
        cn = c.numpy()
        if task.computation is ComputationType.ATB:
            a, b = get_block(task.a_region).numpy(), get_block(task.b_region).numpy()
            if kernel == "naive":
                O.gemm_atb(np.ascontiguousarray(a), np.ascontiguousarray(b), cn, 1.0, count)
            else:
                O.strassen_atb(a, b, cn, 1.0, threshold, count)
            return
        prefix = get_block(task.a_region).numpy()
        s = stripe_split(task)
        d = prefix[:, s:]
        if s > 0:
            if kernel == "naive":
                O.gemm_atb(np.ascontiguousarray(d), np.ascontiguousarray(prefix[:, :s]), cn[:, :s], 1.0, count)
            else:
                O.strassen_atb(d, prefix[:, :s], cn[:, :s], 1.0, threshold, count)
        if kernel == "naive":
            O.syrk_lower(np.ascontiguousarray(d), cn[:, s:], 1.0, count)
        else:
            O.ata_lower(d, cn[:, s:], 1.0, threshold, count)
    return leaf
