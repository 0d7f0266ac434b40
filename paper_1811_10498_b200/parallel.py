"""Multi-GPU text sharding with halo + match-list gather.

One process per GPU.  Rank g owns positions [s_g, e_g) with s_g = align64(g*n/G) and receives the
text [s_g, min(n, e_g + maxlen - 1)) -- the owned range plus a halo of (maxlen - 1) bases, enough for
every walk that starts in the owned range (a walk reads at most maxlen bases; reading R6).
There is no text exchange between GPUs.  The only collectives are the NCCL gathers of the per-rank
match counts and (position, pattern id) lists; rank order is position order, so rank 0 concatenates.
Positions in the lists are global (each rank compacts with pos_base = s_g).
"""
from __future__ import annotations

import dataclasses


@dataclasses.dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int      # s_g, first owned position
    end: int        # e_g, one past the last owned position
    avail_end: int  # one past the last base this rank receives (owned + halo)

    @property
    def n_own(self) -> int:
        return self.end - self.start

    @property
    def n_avail(self) -> int:
        return self.avail_end - self.start


def shard(n: int, world: int, rank: int, maxlen: int, align: int = 64) -> Shard:
    """Contiguous, `align`-aligned shard of [0, n) for `rank` with a (maxlen - 1)-base halo."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")

    def cut(g: int) -> int:
        if g >= world:
            return n
        return min(n, (g * n // world) // align * align)

    s, e = cut(rank), cut(rank + 1)
    halo = max(0, maxlen - 1)
    return Shard(rank, world, s, e, min(n, e + halo) if e > s else e)


def gather_matches(pos, pid, count: int, group=None, dst: int = 0):
    """Gather every rank's first `count` (pos, pid) entries to rank `dst`, in rank order.

    Works for NCCL (CUDA tensors) and gloo (CPU tensors).  Step 1: all_gather of the int64 counts
    (8 B per rank).  Step 2: gather of the lists padded to the largest count (~12 B per match).
    Returns (pos, pid, counts) on `dst` and (None, None, counts) elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo" and pos.is_cuda:  # gloo collectives run on host tensors
        hp, hi, counts = gather_matches(pos[:count].cpu(), pid[:count].cpu(), count, group, dst)
        return (hp.to(pos.device) if hp is not None else None, hi.to(pos.device) if hi is not None else None,
                counts)
    dev = pos.device
    c = torch.tensor([count], dtype=torch.int64, device=dev)
    counts_t = torch.zeros(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(counts_t, c, group=group)
    counts = [int(x) for x in counts_t.cpu().tolist()]
    m = max(counts) if counts else 0
    if m == 0:
        empty = (torch.zeros(0, dtype=pos.dtype, device=dev), torch.zeros(0, dtype=pid.dtype, device=dev))
        return (*empty, counts) if rank == dst else (None, None, counts)
    send_pos = torch.zeros(m, dtype=pos.dtype, device=dev)
    send_pid = torch.zeros(m, dtype=pid.dtype, device=dev)
    send_pos[:count] = pos[:count]
    send_pid[:count] = pid[:count]
    if rank == dst:
        gp = [torch.empty(m, dtype=pos.dtype, device=dev) for _ in range(world)]
        gi = [torch.empty(m, dtype=pid.dtype, device=dev) for _ in range(world)]
    else:
        gp = gi = None
    dist.gather(send_pos, gp, dst=dst, group=group)
    dist.gather(send_pid, gi, dst=dst, group=group)
    if rank != dst:
        return None, None, counts
    return (torch.cat([g[:k] for g, k in zip(gp, counts)]), torch.cat([g[:k] for g, k in zip(gi, counts)]),
            counts)


# ----------------------------------------------------------------------------- sync-free gather
def list_buffer(cap: int, device):
    """One byte buffer holding a rank's whole result, [count int64 | pos int64[cap] | pid int32[cap]]
    (padded to 16 B), and its (count, pos, pid) views: the match kernels write straight into it, and
    one gather moves it -- no host read of the count inside a step."""
    import torch
    nbytes = (8 + 12 * cap + 15) // 16 * 16
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    count = buf[0:8].view(torch.int64)
    pos = buf[8:8 + 8 * cap].view(torch.int64)
    pid = buf[8 + 8 * cap:8 + 12 * cap].view(torch.int32)
    return buf, count, pos, pid


def gather_lists_async(buf, group=None, dst: int = 0):
    """Gather every rank's list buffer (list_buffer) to rank `dst`: one NCCL gather of fixed-size
    buffers, stream-ordered after the kernel that filled them (no host synchronisation).  Returns a
    (world, nbytes) uint8 tensor on `dst`, None elsewhere.  gloo: staged through host memory."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    src = buf.cpu() if (dist.get_backend(group) == "gloo" and buf.is_cuda) else buf
    out = torch.empty((world, src.numel()), dtype=torch.uint8, device=src.device) if rank == dst else None
    dist.gather(src, list(out.unbind(0)) if out is not None else None, dst=dst, group=group)
    if out is not None and out.device != buf.device:
        out = out.to(buf.device)
    return out


def unpack_lists(gathered, cap: int):
    """Rank-order concatenation of gathered list buffers: (pos int64, pid int32, counts).  Counts
    above `cap` (a rank's list overflowed its buffer) raise: the caller must re-run with a larger cap."""
    import torch
    g = gathered.cpu()
    counts = [int(x) for x in g[:, 0:8].contiguous().view(torch.int64).flatten().tolist()]
    if any(c > cap for c in counts):
        raise ValueError(f"a rank's match count exceeds the list capacity {cap}: {counts}")
    pos = [g[r, 8:8 + 8 * cap].contiguous().view(torch.int64)[:c] for r, c in enumerate(counts)]
    pid = [g[r, 8 + 8 * cap:8 + 12 * cap].contiguous().view(torch.int32)[:c] for r, c in enumerate(counts)]
    return torch.cat(pos), torch.cat(pid), counts


# ----------------------------------------------------------------------------- one rank's step
class ShardedMatcher:
    """One rank's part of the N-GPU hot path.

    The rank holds its text shard (owned positions + a (maxlen - 1)-base halo, `Shard`) on its GPU.
    A step is the text call -- pack + match + compact in one kernel (pfac_match_text_async) -- with
    pos_base = s_g, writing the count and the (position, pattern id) list straight into the rank's
    list buffer, followed (N > 1) by one gather of the fixed-size buffers to `dst`.  No text moves
    between GPUs; the only collective is the gather (rank order = position order).

    cap: list capacity, the same on every rank (see `agree_capacity`).  dense_out: also write the
    dense out[] of the owned positions (the paper's output array).
    """

    def __init__(self, a, d_text, sh: Shard, cap: int, dense_out: bool = True, group=None, dst: int = 0):
        import torch

        from . import binding as B
        self.a, self.d_text, self.sh, self.cap, self.group, self.dst = a, d_text, sh, cap, group, dst
        dev = d_text.device
        self.buf, self.count, self.pos, self.pid = list_buffer(cap, dev)
        self.out = torch.empty(max(sh.n_own, 1), dtype=torch.int32, device=dev)[:sh.n_own] if dense_out else None
        self.ws = torch.empty(B.match_text_workspace_bytes(sh.n_own, sh.n_avail, not dense_out), dtype=torch.uint8,
                              device=dev)
        self.first_bad = torch.zeros(1, dtype=torch.int64, device=dev)

    def match(self, stream=None) -> None:
        """The rank's text call (asynchronous on `stream`)."""
        from . import binding as B
        B.match_text_async(self.a, self.d_text, self.sh.n_own, self.sh.n_avail, self.out, self.pos, self.pid,
                           self.count, self.ws, pos_base=self.sh.start, first_bad=self.first_bad, stream=stream)

    def gather(self):
        """gather_lists_async of this rank's buffer: (world, nbytes) on dst, None elsewhere."""
        return gather_lists_async(self.buf, group=self.group, dst=self.dst)

    def step(self, stream=None):
        self.match(stream)
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            return self.gather()
        return None


def probe_count(a, d_text, sh: Shard) -> int:
    """The exact match count of this rank's shard (a capacity-0 text call; synchronous)."""
    import torch

    from . import binding as B
    dev = d_text.device
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    empty64 = torch.empty(1, dtype=torch.int64, device=dev)[:0]
    empty32 = torch.empty(1, dtype=torch.int32, device=dev)[:0]
    ws = torch.empty(B.match_text_workspace_bytes(sh.n_own, sh.n_avail, True), dtype=torch.uint8, device=dev)
    B.match_text_async(a, d_text, sh.n_own, sh.n_avail, None, empty64, empty32, cnt, ws, pos_base=sh.start)
    return int(cnt.item())


def agree_capacity(local_count: int, group=None, slack: int = 1024) -> int:
    """One list capacity for every rank: the largest rank's count + slack (all_reduce MAX; outside
    the timed region).  gloo reduces on the host, NCCL on the device."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local_count + slack
    dev = "cpu" if dist.get_backend(group) == "gloo" else torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([local_count + slack], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())
