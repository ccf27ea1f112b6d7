"""Graph-CoT multi-agent workload driver over the engine (the caller side of the hot path).

Mirrors the reference's Orchestrator state machine in GLM mode (orchestrator.cpp:156-256) with a
scripted provider (scripted.hpp:21-30) whose replies follow the Rule agent's formats
(rule.cpp:156-236) and run_bench's deterministic round-robin (bench.cpp:65-83):

  Classifying -> "no"                                   (classification prompt)
  Reasoning   -> "Missing: vertex chunks for: <id_r>"   (reasoning prompt: notebook = tier II)
  Acting      -> fenced print(NodeInfo(RetrieveNode("<id_r>")))   (action prompt)
                 the snippet output (K1 vertex chunk + "\\n") is appended to the notebook
  ... one source node per round, then Reasoning -> "Finish: <answer>" and
  finish(): set_tier(session, II, III) (orchestrator.cpp:147-154).

One rotation = every active lane makes its next LLM call; the rotation's calls are ONE engine
prefill batch (bookkeeping applied in lane order, as the reference would), and ONE batched K1
launch builds the vertex chunks of every action executed in that rotation, overlapped with the
prefill on the graph's stream.  Source nodes are
drawn with a power-law skew so popular (hub) chunks recur across queries; every reasoning round
re-reads the previous rounds' chunks (reuse across iterations).
"""
from __future__ import annotations

import ctypes as C
import random
import threading
from dataclasses import dataclass, field

from . import _lib, synth
from ._lib import check, lib
from .kvcache import PrefillReport, count_tokens  # noqa: F401  (count_tokens: tokenizer.hpp:36-46)
from .templates import TIER_II, TIER_III, TIER_IV, TemplateSet


@dataclass
class Session:
    sid: str
    sources: list
    question: str
    state: str = "C"
    round: int = 0
    notebook: str = ""
    calls: int = 0
    task: str = ""


@dataclass
class Call:
    session: Session
    agent: str
    segments: list
    reply: str

    @property
    def is_finish(self):
        return self.agent == "reasoning" and self.reply.startswith("Finish:")


@dataclass
class RotationResult:
    calls: int = 0
    prompt_tokens: int = 0       # cached + computed + tail
    computed_tokens: int = 0     # computed + tail (what the GPU ran)
    cached_tokens: int = 0
    finished: int = 0
    chunks: int = 0
    chunk_bytes: int = 0         # K1 algorithmic bytes (CSR rows, neighbour pairs, entries, out)
    chunk_ms: float = 0.0        # K1 device time of this rotation's chunk build
    retrieve_ms: float = 0.0     # K5 device time (0 when every RetrieveNode hit the LRU)
    retrieve_probes: int = 0     # index probes (LRU misses) of this rotation
    decoded_tokens: int = 0      # reply tokens decoded after the prefill (rotation_with_decode)
    decode_collected: bool = True  # False: this rotation's decode was deferred into the next
    reports: list = field(default_factory=list)
    first_tokens: list = field(default_factory=list)
    calls_made: list = field(default_factory=list)  # the rotation's Calls, in lane order


class GraphCoTWorkload:
    def __init__(self, engine, retriever, n_queries, lanes, seed=0, min_hops=2, max_hops=4,
                 skew=2.5, templates=None, node_ids=None, overlap_retrieval=True,
                 question_pool=0, node_index=None, repeat_frac=0.0, repeat_window=256):
        self.engine = engine
        # node_index (NodeIndex): the action's RetrieveNode("<id>") is resolved by the K5 nearest
        # scan + retrieval LRU (retriever.cpp:49-66) instead of taking the scripted source node
        self.node_index = node_index
        self.overlap_retrieval = overlap_retrieval
        self.kv = engine.kv if engine is not None else None
        self.retriever = retriever
        self.templates = templates or TemplateSet()
        self.lanes = lanes
        g = retriever.graph
        # the question stream (synth.graph_cot_questions, shared with bench.py's reference arm);
        # question_pool > 0: questions are drawn WITH replacement from that many candidate source
        # lists, as generate_workload picks clusters (workload.cpp:216-225), so questions recur
        # across sessions (and, sharded i mod N, across GPUs)
        self.sessions = []
        for sid, src, _ in synth.graph_cot_questions(g.node_count(), n_queries, seed, min_hops,
                                                     max_hops, skew, question_pool, repeat_frac,
                                                     repeat_window):
            ids = [g.node_id(v) for v in src]
            question = "Which item is linked from all of: " + "; ".join(ids) + "?"
            self.sessions.append(Session(sid, src, question))
        self.admitted = 0
        self.active = []

    def done(self):
        return self.admitted >= len(self.sessions) and not self.active

    def _call_for(self, s: Session) -> Call:
        t = self.templates
        if s.state == "C":
            return Call(s, "classification", t.render_classification(s.question),
                        synth.classify_reply())
        if s.state == "R":
            if s.round < len(s.sources):
                nid = self.retriever.graph.node_id(s.sources[s.round])
                s.task = "vertex chunks for: " + nid
                return Call(s, "reasoning", t.render_reasoning(s.question, s.notebook),
                            synth.missing_reply(nid))
            return Call(s, "reasoning", t.render_reasoning(s.question, s.notebook),
                        synth.finish_reply(self.retriever.graph.node_id(s.sources[0])))
        nid = s.task[len("vertex chunks for: "):]
        return Call(s, "action", t.render_action(s.task), synth.action_reply(nid))

    def next_calls(self):
        """Admission + one call per active lane, in lane order (bench.cpp:71-76)."""
        while len(self.active) < self.lanes and self.admitted < len(self.sessions):
            self.active.append(self.sessions[self.admitted])
            self.admitted += 1
        return [self._call_for(s) for s in self.active]

    @staticmethod
    def pack(calls):
        n = len(calls)
        arr = (_lib.SegmentRequestC * max(1, n))()
        keep = []
        for i, c in enumerate(calls):
            texts = [txt.encode() for _, txt in c.segments]
            ta = (C.c_char_p * max(1, len(texts)))(*texts)
            la = (C.c_uint64 * max(1, len(texts)))(*[len(x) for x in texts])
            tr = (C.c_int32 * max(1, len(texts)))(*[t for t, _ in c.segments])
            sb = c.session.sid.encode()
            keep += [texts, ta, la, tr, sb]
            arr[i].seg_text, arr[i].seg_len, arr[i].seg_tier = ta, la, tr
            arr[i].n_seg, arr[i].session = len(texts), sb
            # a Finish reply: Orchestrator::finish's set_tier(II -> III) follows this call's
            # bookkeeping inside the batch, before the next lane's (run_bench order)
            arr[i].finish = int(c.is_finish)
        return arr, keep

    def prefill(self, calls, packed=None):
        n = len(calls)
        arr, keep = packed if packed is not None else self.pack(calls)
        reps = (_lib.PrefillReportC * max(1, n))()
        first = (C.c_int32 * max(1, n))()
        check(lib().glmx_engine_prefill_segments(self.engine.h, n, arr, reps, first, None))
        return ([PrefillReport(reps[i].cached_tokens, reps[i].computed_tokens,
                               reps[i].tail_tokens) for i in range(n)], [first[i] for i in range(n)])

    def advance(self, calls, reports=None, first_tokens=None, chunks=None) -> RotationResult:
        """Apply the replies: state transitions, K1 chunk build for the actions (or the batch
        `chunks` already built for them), finish."""
        res = RotationResult(calls=len(calls), reports=reports or [],
                             first_tokens=first_tokens or [], calls_made=list(calls))
        for r in res.reports:
            res.cached_tokens += r.cached_tokens
            res.computed_tokens += r.computed_tokens + r.tail_tokens
            res.prompt_tokens += r.cached_tokens + r.computed_tokens + r.tail_tokens
        acting = [c for c in calls if c.agent == "action"]
        if acting:
            batch = chunks if chunks is not None else self._retrieve_and_build(acting)
            for c, text in zip(acting, batch.texts):
                c.session.notebook += text + "\n"  # PrintStmt: raw chunk + "\n" (interp.cpp:68-74)
            res.chunks = len(acting)
            res.chunk_ms = batch.kernel_ms
            res.retrieve_ms = getattr(batch, "retrieve_ms", 0.0)
            res.retrieve_probes = getattr(batch, "retrieve_probes", 0)
            g = self.retriever.graph
            res.chunk_bytes = sum(8 + 8 * g.total_degree(v) for v in batch.nodes)
            res.chunk_bytes += sum(2 * len(t) + 20 * len(sp) for t, sp in
                                   zip(batch.texts, batch.token_spans))
        still = []
        for c in calls:
            s = c.session
            s.calls += 1
            if c.agent == "classification":
                s.state = "R"
            elif c.agent == "action":
                s.round += 1
                s.state = "R"
            elif c.is_finish:  # set_tier(II -> III) ran inside the prefill batch (pack)
                s.state = "done"
                res.finished += 1
                continue
            else:
                s.state = "A"
            still.append(s)
        self.active = still
        return res

    def _retrieve_and_build(self, acting):
        """RetrieveNode (K5, when a node index is attached) then NodeInfo chunks (K1) for the
        rotation's action snippets; both on the graph's stream."""
        probes0 = probes1 = 0
        r_ms = 0.0
        if self.node_index is not None:
            texts = [c.session.task[len("vertex chunks for: "):] for c in acting]
            probes0 = self.node_index.stats()[2]
            nodes, _ = self.node_index.retrieve_nodes(texts)
            probes1 = self.node_index.stats()[2]
            r_ms = self.node_index.last_kernel_ms() if probes1 > probes0 else 0.0
        else:
            nodes = [c.session.sources[c.session.round] for c in acting]
        batch = self.retriever.chunk_build(nodes)
        batch.nodes = nodes
        batch.retrieve_ms = r_ms
        batch.retrieve_probes = probes1 - probes0
        return batch

    def prefill_async(self, calls):
        """Bookkeeping + staging now (reports returned), forward enqueued; see wait()."""
        n = len(calls)
        arr, keep = self.pack(calls)
        reps = (_lib.PrefillReportC * max(1, n))()
        check(lib().glmx_engine_prefill_segments_async(self.engine.h, n, arr, reps))
        del keep  # the call tokenised the segments before returning
        return [PrefillReport(reps[i].cached_tokens, reps[i].computed_tokens, reps[i].tail_tokens)
                for i in range(n)]

    def wait(self, n):
        """Completes the oldest in-flight batch; its greedy first tokens."""
        first = (C.c_int32 * max(1, n))()
        m = lib().glmx_engine_wait(self.engine.h, first, max(1, n))
        if m < 0:
            check(-m)
        return [first[i] for i in range(n)]

    def _start_retrieval(self, calls):
        acting = [c for c in calls if c.agent == "action"]
        built = {}
        th = None
        if acting:
            th = threading.Thread(target=lambda: built.__setitem__(
                "b", self._retrieve_and_build(acting)))
            th.start()
        return th, built

    def rotations(self, count, peer=None):
        """`count` rotations, pipelined: the host work of rotation r+1 (its calls, the
        bookkeeping and staging of its prefill, its RetrieveNode/K1 thread) runs while rotation
        r's forward is on the GPU.  Nothing host-side depends on a forward's output (replies are
        scripted), and the engine stream orders the forwards, so the cache decisions and the
        results are those of the sequential loop.  Yields each rotation's RotationResult after its
        forward completed (engine timings/work then describe that rotation).

        peer: a sharding.PeerExchange running the pipelined epoch protocol (before_bookkeeping
        ahead of every prefill, after_wait behind every completed forward) for multi-GPU runs."""
        if count <= 0:
            return
        calls = self.next_calls()
        th, built = self._start_retrieval(calls)
        if peer is not None:
            peer.before_bookkeeping()
        reps = self.prefill_async(calls)
        for r in range(count):
            if th is not None:
                th.join()
            res = self.advance(calls, reps, None, chunks=built.get("b"))
            nxt = None
            if r + 1 < count:
                calls_n = self.next_calls()
                th_n, built_n = self._start_retrieval(calls_n)
                if peer is not None:
                    peer.before_bookkeeping()
                nxt = (calls_n, th_n, built_n, self.prefill_async(calls_n))
            res.first_tokens = self.wait(len(calls))
            if peer is not None:
                peer.after_wait()
            yield res
            if nxt is not None:
                calls, th, built, reps = nxt

    def rotation_with_decode(self, max_decode) -> RotationResult:
        """A rotation whose calls are completed like call_llm's provider step: after the prefill
        (which yields each reply's first token) every call greedily decodes the rest of its reply,
        tokens_out - 1 tokens (tokens_out = count_tokens(reply), finalize_completion
        provider.cpp:12-29), capped at max_decode.  The scripted reply text still drives the
        state machine."""
        calls = self.next_calls()
        steps = [max(0, min(max_decode, count_tokens(c.reply) - 1)) for c in calls]
        acting = [c for c in calls if c.agent == "action"]
        th, built = self._start_retrieval(calls) if self.overlap_retrieval else (None, {})
        try:
            reps, first = self.prefill(calls)
        finally:
            if th is not None:
                th.join()
        self.last_prefill_forward_ms = self.engine.last_timings()["forward"]
        if any(steps):
            self.engine.decode(steps)
        res = self.advance(calls, reps, first, chunks=built.get("b") if acting else None)
        res.decoded_tokens = sum(steps)
        return res

    def rotations_with_decode(self, count, max_decode, peer=None, merge=False):
        """`count` rotations of rotation_with_decode, pipelined on one engine stream: the GPU
        runs prefill r, decode r, prefill r+1, decode r+1, ... back to back while the host
        advances the state machines with r's (scripted) replies and stages rotation r+1's prefill
        (bookkeeping, staging, RetrieveNode/K1) before r's decode has finished
        (glmx_engine_decode_async / _collect; the engine stages decode steps and prefills in a
        ring of pinned slots).  Cache decisions and tokens are those of the sequential loop.
        Yields each rotation's RotationResult; engine.last_timings() then holds the last
        collected decode and self.last_prefill_forward_ms the prefill.

        merge: continuous batching of the decode rows of two consecutive rotations (even
        rotations defer their decode into the next one's: one weight stream per decode step for
        both; replies are scripted, so no call waits on them).
        peer: a sharding.PeerExchange running the pipelined epoch protocol (as in rotations())."""
        if count <= 0:
            return

        def steps_of(calls):
            return [max(0, min(max_decode, count_tokens(c.reply) - 1)) for c in calls]

        state = {"deferred": False}
        self.decode_log = []  # (rotation, per-call decoded tokens) in collect order

        def launch_decode(r, steps):
            """Right after rotation r's prefill is staged; True if a decode was enqueued."""
            if merge and not state["deferred"] and r + 1 < count and any(steps):
                self.engine.decode_defer(steps)
                state["deferred"] = True
                return False
            if any(steps) or state["deferred"]:
                self.engine.decode_async(steps)
                state["deferred"] = False
                return True
            return False

        calls = self.next_calls()
        th, built = self._start_retrieval(calls) if self.overlap_retrieval else (None, {})
        if peer is not None:
            peer.before_bookkeeping()
        reps = self.prefill_async(calls)
        steps = steps_of(calls)
        enq = launch_decode(0, steps)
        for r in range(count):
            if th is not None:
                th.join()
            acting = [c for c in calls if c.agent == "action"]
            res = self.advance(calls, reps, None, chunks=built.get("b") if acting else None)
            res.decoded_tokens = sum(steps)
            nxt = None
            if r + 1 < count:
                calls_n = self.next_calls()
                th_n, built_n = (self._start_retrieval(calls_n) if self.overlap_retrieval
                                 else (None, {}))
                if peer is not None:
                    peer.before_bookkeeping()
                nxt = (calls_n, th_n, built_n, self.prefill_async(calls_n), steps_of(calls_n))
            res.first_tokens = self.wait(len(calls))
            if peer is not None:
                peer.after_wait()
            self.last_prefill_forward_ms = self.engine.last_timings()["forward"]
            res.decode_collected = enq
            if enq:
                cur, prev = self.engine.decode_collect()
                if prev is not None:
                    self.decode_log.append((r - 1, prev))
                self.decode_log.append((r, cur))
            yield res
            if nxt is not None:
                calls, th, built, reps, steps = nxt
                enq = launch_decode(r + 1, steps)

    def rotation(self) -> RotationResult:
        """One round-robin rotation.  The actions' RetrieveNode -> NodeInfo chunks depend only on
        the (scripted) action code, not on this prefill, so K1 runs on the graph's own CUDA stream
        in a second host thread while the prefill batch runs on the engine stream (the GIL is
        released inside both C-ABI calls); the chunk texts join the notebooks afterwards, exactly
        where the sequential order puts them."""
        calls = self.next_calls()
        acting = [c for c in calls if c.agent == "action"]
        built = {}
        th = None
        if acting and self.overlap_retrieval:
            th = threading.Thread(target=lambda: built.__setitem__(
                "b", self._retrieve_and_build(acting)))
            th.start()
        try:
            reps, first = self.prefill(calls)
        finally:
            if th is not None:
                th.join()
        return self.advance(calls, reps, first, chunks=built.get("b"))


def adversarial_priority_ops(n_hot=8, rounds=12, n_cold=24, notebook_words=240, cold_words=300,
                             seed=0):
    """The priority-vs-LRU adversarial stream SPEC.md:532/778 asks for (the reference ships
    none): n_hot reasoning sessions whose prompts re-read a long retrieved-chunk notebook
    (tier II) every round, separated by floods of one-off agent prompts (tier IV: transient
    task/question text, never reused).  Sized by the caller's capacity so that the hot notebooks
    fit but hot + one flood do not: plain LRU evicts the notebooks during every flood (they are
    the least recently used), four-tier priority evicts the tier-IV flood first and keeps them.

    Returns the op list [("p", (tokens, tiers), session), ...] in the reference's prefill terms
    (templates render_reasoning: tier I instructions, tier II notebook, tier IV question)."""
    rnd = random.Random(seed)
    t = TemplateSet()
    vocab = [f"w{rnd.randrange(10**6)}" for _ in range(4096)]
    notebooks = [" ".join(rnd.choice(vocab) for _ in range(notebook_words)) for _ in range(n_hot)]
    questions = [f"Which item is linked from all of: h{h}a; h{h}b?" for h in range(n_hot)]
    ops = []
    for r in range(rounds):
        for h in range(n_hot):
            segs = t.render_reasoning(questions[h], notebooks[h])
            ops.append(("p", segs, f"hot{h}"))
        for c in range(n_cold):
            text = " ".join(rnd.choice(vocab) for _ in range(cold_words))
            ops.append(("p", [(TIER_IV, f"r{r}c{c} " + text)], f"cold{r}_{c}"))
    return ops
