"""PromptTemplate (prompt.cpp) and SlotPlan (router.cpp) restated.

Test infrastructure only.  Actions are tuples ``(kind, start, tokens)`` with
kind in {"prefill_only", "generate", "reclaim"} (router.hpp:11-17).
"""
from __future__ import annotations

from .topology import RunError, ValidationError, aid


class PromptTemplate:
    """prefix ++ (sep_1 ++ out_1) ++ ... ++ suffix (prompt.hpp:27-53)."""

    def __init__(self, prefix, slots, suffix):
        # slots: list of (precursor, separator)
        seen = set()
        for p, _ in slots:
            if p in seen:  # prompt.cpp:8-17
                raise ValidationError(f"prompt template: precursor {aid(p)} appears in more than one slot")
            seen.add(p)
        self.prefix = list(prefix)
        self.slots = [(p, list(s)) for p, s in slots]
        self.suffix = list(suffix)

    def without(self, pruned):
        """prompt.cpp:26-37."""
        kept = [(p, s) for p, s in self.slots if p != pruned]
        if len(kept) == len(self.slots):
            raise ValidationError(f"prompt template: cannot drop {aid(pruned)}; it has no slot")
        return PromptTemplate(self.prefix, kept, self.suffix)


def assemble(tmpl: PromptTemplate, outputs: dict) -> list:
    """prompt.cpp:47-78 (tokens only)."""
    out = list(tmpl.prefix)
    for p, sep in tmpl.slots:
        if p not in outputs:
            raise ValidationError(f"assemble: missing output for precursor {aid(p)}")
        out += sep
        out += outputs[p]
    out += tmpl.suffix
    return out


class _Slot:
    __slots__ = ("precursor", "separator", "received", "issued", "sep_issued", "closed", "mark", "phase")

    def __init__(self, p, sep):
        self.precursor, self.separator = p, list(sep)
        self.received, self.issued, self.sep_issued, self.closed, self.mark = [], 0, False, False, 0
        self.phase = "waiting"


class SlotPlan:
    """Slot-filling shell router (router.cpp:9-184)."""

    def __init__(self, self_id, tmpl: PromptTemplate, incremental: bool):
        self.self_id, self.tmpl, self.incremental = self_id, tmpl, incremental
        self.slots = [_Slot(p, s) for p, s in tmpl.slots]
        self.had_slots = bool(self.slots)
        self.started = False
        self.active = 0
        self.suffix_issued = False
        self.scheduled = 0
        self.calls = 0
        self.reclaims = 0
        self.pending = []
        self.issued_stream = []
        self.generate_issued = False
        self.final_prompt = None

    def all_inputs_pruned(self):
        return self.had_slots and not self.slots

    def _idx(self, producer):
        for i, s in enumerate(self.slots):
            if s.precursor == producer:
                return i
        return -1

    def outputs(self):
        return {s.precursor: list(s.received) for s in self.slots}

    def start(self):
        """router.cpp:38-42."""
        if self.started:
            raise RunError(f"router: started twice for agent {aid(self.self_id)}")
        self.started = True
        return self._advance()

    def on_chunk(self, producer, tokens):
        """router.cpp:44-55."""
        i = self._idx(producer)
        if i < 0:
            return []
        if self.generate_issued:
            raise RunError(f"router: chunk from {aid(producer)} after generate for {aid(self.self_id)}")
        s = self.slots[i]
        if s.closed:
            raise RunError(f"router: chunk after stream close from {aid(producer)}")
        s.received += list(tokens)
        if not self.started:
            return []
        return self._advance()

    def on_precursor_done(self, producer):
        """router.cpp:57-64."""
        i = self._idx(producer)
        if i < 0:
            return []
        self.slots[i].closed = True
        if not self.started:
            return []
        return self._advance()

    def on_precursor_cancelled(self, producer):
        """router.cpp:66-99."""
        i = self._idx(producer)
        if i < 0:
            return []
        if self.generate_issued:
            raise RunError(f"router: precursor {aid(producer)} pruned after generate for {aid(self.self_id)}")
        if i < self.active:
            raise RunError(f"router: completed precursor {aid(producer)} cannot be pruned")
        actions = []
        if i == self.active:
            s = self.slots[i]
            if s.sep_issued and self.scheduled > s.mark:
                actions.append(("reclaim", s.mark, []))
                self.reclaims += 1
                self.scheduled = s.mark
                del self.issued_stream[s.mark:]
        self.tmpl = self.tmpl.without(producer)
        del self.slots[i]
        if not self.started:
            return actions
        return actions + self._advance()

    def _flush(self, out):
        """router.cpp:101-112."""
        if not self.pending:
            return
        toks = self.pending
        self.pending = []
        out.append(("prefill_only", self.scheduled, toks))
        self.scheduled += len(toks)
        self.issued_stream += toks
        self.calls += 1

    def _advance(self):
        """router.cpp:114-184."""
        actions = []
        if self.generate_issued:
            return actions
        if not self.incremental:
            if any(not s.closed for s in self.slots):
                return actions
            self.final_prompt = assemble(self.tmpl, self.outputs())
            actions.append(("generate", 0, list(self.final_prompt)))
            self.generate_issued = True
            return actions
        if self.scheduled == 0 and not self.pending and self.active == 0:
            self.pending += self.tmpl.prefix
        progressed = True
        while progressed:
            progressed = False
            if self.active < len(self.slots):
                s = self.slots[self.active]
                if not s.sep_issued:
                    s.mark = self.scheduled + len(self.pending)
                    self.pending += s.separator
                    s.sep_issued = True
                    s.phase = "filling"
                if s.issued < len(s.received):
                    self.pending += s.received[s.issued:]
                    s.issued = len(s.received)
                if s.closed and s.issued == len(s.received):
                    s.phase = "complete"
                    self.active += 1
                    progressed = True
        if self.active == len(self.slots):
            if not self.suffix_issued:
                self.pending += self.tmpl.suffix
                self.suffix_issued = True
            self._flush(actions)
            assembled = assemble(self.tmpl, self.outputs())
            if assembled != self.issued_stream:
                raise RunError(f"router: issued prompt diverged from template assembly for {aid(self.self_id)}")
            self.final_prompt = assembled
            actions.append(("generate", 0, list(assembled)))
            self.generate_issued = True
            return actions
        self._flush(actions)
        return actions
