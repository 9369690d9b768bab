"""Execution traces and the communication cost model of the sharded solve
(SURVEY.md 8f row f4).

Mirrors the reporting half of the reference's virtual harness
(``harness.py:45-89`` ExecutionTrace, ``harness.py:236-304`` cost model and
``audit_trace``) for the real multi-GPU path in :mod:`.distributed`:

* On NVSwitch one NCCL all-gather replaces the reference's dissemination
  rounds.  :func:`allgather_schedule` writes the LOGICAL dissemination
  schedule of an all-gather of equal per-rank payloads into an
  :class:`ExecutionTrace` -- stage s: rank r sends the window of
  min(2^s, W - 2^s) slots starting at its own to rank (r - 2^s) mod W,
  chunked so no message exceeds the per-message cap.  Fed the reference's own
  protocol (P slots of one (base, carry) pair, cap M^2 + M doubles per RHS) it
  reproduces the reference harness trace record for record
  (tests/test_trace.py pins this against a trace the reference wrote).
* :class:`ShardedPlan <.distributed.ShardedPlan>` records its two per-solve
  all-gathers (carry blocks, crossing-node partial sums) this way when given a
  trace, plus the measured time of each collective (CUDA events on the NCCL
  stream; wall clock for gloo).  Its stage count is therefore
  ``collectives * ceil(log2 W)`` with W = GPUs, not the reference's
  ``ceil(log2 P)`` over P virtual ranks; :func:`audit_trace` takes the
  number of collectives.
"""

from __future__ import annotations

import io as _io
import math

from . import errors as _err


class ExecutionTrace:
    """Ordered per-stage message log (ref harness.py:45-89): (stage, sender, receiver, nbytes)."""

    def __init__(self, nranks):
        self.nranks = nranks
        self.records = []
        self.timings = []  # (label, milliseconds) of the real collectives behind the logical stages

    def add(self, stage, msg_or_sender, receiver=None, nbytes=None):
        if receiver is None:  # a Message-like object (sender, receiver, nbytes)
            m = msg_or_sender
            self.records.append((stage, m.sender, m.receiver, m.nbytes))
        else:
            self.records.append((stage, msg_or_sender, receiver, nbytes))

    @property
    def stages(self) -> int:
        return max((r[0] for r in self.records), default=-1) + 1

    def per_rank_stages(self):
        active = [set() for _ in range(self.nranks)]
        for stage, snd, rcv, _ in self.records:
            active[snd].add(stage)
            active[rcv].add(stage)
        return [len(s) for s in active]

    def stage_rank_bytes(self):
        out = {}
        for stage, snd, _, nbytes in self.records:
            out[(stage, snd)] = out.get((stage, snd), 0) + nbytes
        return out

    def max_message_bytes(self) -> int:
        return max((r[3] for r in self.records), default=0)

    def total_bytes(self) -> int:
        return sum(r[3] for r in self.records)

    def to_csv(self, path=None):
        buf = _io.StringIO()
        buf.write("stage,sender,receiver,bytes\n")
        for rec in self.records:
            buf.write("%d,%d,%d,%d\n" % rec)
        text = buf.getvalue()
        if path is not None:
            with open(path, "w") as fh:
                fh.write(text)
        return text


def allgather_schedule(trace, nranks, slot_bytes, cap_bytes, stage0=0):
    """Append the dissemination schedule of an all-gather of one ``slot_bytes``
    payload per rank (ceil(log2 nranks) stages from ``stage0``).  Messages carry
    whole slots up to ``cap_bytes``; a slot larger than the cap is split into
    cap-sized pieces.  Returns the number of stages written."""
    rounds = (nranks - 1).bit_length()
    per_msg = max(1, cap_bytes // slot_bytes) if slot_bytes else 1
    for s in range(rounds):
        shift = 1 << s
        count = min(shift, nranks - shift)
        for r in range(nranks):
            dest = (r - shift) % nranks
            for ofs in range(0, count, per_msg):
                c = min(per_msg, count - ofs)
                nbytes = c * slot_bytes
                if slot_bytes > cap_bytes > 0:
                    while nbytes > 0:
                        piece = min(cap_bytes, nbytes)
                        trace.add(stage0 + s, r, dest, piece)
                        nbytes -= piece
                else:
                    trace.add(stage0 + s, r, dest, nbytes)
    return rounds


def reference_protocol_trace(p, m, nrhs):
    """The reference harness's per-solve trace (harness.py:147-216) for P = p
    virtual ranks: all-gather of one (base, carry) pair (2 M K doubles) per rank,
    at most max(1, (M^2 + M) // (2M)) pairs per message."""
    tr = ExecutionTrace(p)
    slot = 2 * m * nrhs * 8
    allgather_schedule(tr, p, slot, max(1, (m * m + m) // (2 * m)) * slot)
    return tr


class CostModelParams:
    """alpha [s], beta [s/byte], block order m, ranks p (ref harness.py:236-247)."""

    __slots__ = ("alpha", "beta", "m", "p")

    def __init__(self, alpha, beta, m, p):
        if alpha < 0 or beta < 0:
            raise ValueError("alpha and beta must be nonnegative")
        self.alpha, self.beta, self.m, self.p = float(alpha), float(beta), int(m), int(p)


def predict_preprocess_comm(params: CostModelParams) -> float:
    """alpha log2 p + p/(p-1) beta M^2 (ref harness.py:250-257)."""
    if params.p < 2:
        raise _err.InvalidRankCount("communication model needs p >= 2")
    return params.alpha * math.log2(params.p) + params.p / (params.p - 1) * params.beta * params.m ** 2


def predict_solve_comm(params: CostModelParams) -> float:
    """alpha log2^2 p + 4 M^2 log2(p) beta (ref harness.py:260-266)."""
    if params.p < 2:
        raise _err.InvalidRankCount("communication model needs p >= 2")
    lg = math.log2(params.p)
    return params.alpha * lg * lg + 4.0 * params.m ** 2 * lg * params.beta


def audit_trace(trace: ExecutionTrace, params: CostModelParams, nrhs: int = 1, collectives: int = 1):
    """Check the stage structure of a solve trace and price it (ref harness.py:269-304).

    Expects exactly ``collectives * ceil(log2 p)`` stages (the reference's
    protocol has one collective; the sharded GPU solve has two when tree nodes
    cross rank boundaries) and no message above (M^2 + M) * nrhs doubles.
    ``trace_model_seconds`` prices the trace as sum over stages of
    alpha + beta * (max bytes any rank sends in that stage)."""
    expected = collectives * (math.ceil(math.log2(params.p)) if params.p > 1 else 0)
    stages = trace.stages
    if stages != expected:
        raise _err.StageViolation(f"trace has {stages} stages, expected {expected}")
    cap = (params.m ** 2 + params.m) * 8 * nrhs
    worst = trace.max_message_bytes()
    if worst > cap:
        raise _err.StageViolation(f"message of {worst} bytes exceeds cap {cap}")
    per_stage = [0] * stages
    for (stage, _rank), nbytes in trace.stage_rank_bytes().items():
        per_stage[stage] = max(per_stage[stage], nbytes)
    trace_model = sum(params.alpha + params.beta * h for h in per_stage)
    model = predict_solve_comm(params) if params.p >= 2 else 0.0
    return {
        "stages": stages,
        "max_message_bytes": worst,
        "max_stage_rank_bytes": max(per_stage, default=0),
        "total_bytes": trace.total_bytes(),
        "trace_model_seconds": trace_model,
        "predict_solve_seconds": model,
        "model_residual": trace_model - model,
        "measured_ms": [ms for _label, ms in trace.timings],
    }


__all__ = ["CostModelParams", "ExecutionTrace", "allgather_schedule", "audit_trace", "predict_preprocess_comm",
           "predict_solve_comm", "reference_protocol_trace"]
