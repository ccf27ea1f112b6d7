"""Reference-trace driver: the reference's Orchestrator in GLM mode (orchestrator.cpp:156-330)
with its ScriptedProvider (scripted.hpp:12-30, provider.cpp:31-62) and run_bench's deterministic
round-robin (bench.cpp:65-83), over the engine.  This is configuration C1 end to end: the
reference's own prompt templates and notebook produce the segments, K5 resolves RetrieveNode, K1
builds the NodeInfo vertex chunks, the engine runs the prefill (bookkeeping + forward) and the
greedy decode of every reply.

Per rotation every active session makes its next call, in lane order.  The calls of a rotation
are ONE engine prefill batch: the engine applies the bookkeeping request by request in lane
order, and a call whose reply is Finish carries the `finish` flag, so Orchestrator::finish's
set_tier(II -> III) (orchestrator.cpp:147-154) lands right after that call's prefill, exactly
where the reference's run_step puts it.  Replies are scripted, so they are known before the
prefill; the decoded tokens (random-init weights) do not drive control flow, the script does.

Action snippets: the snippet interpreter is out of scope.  This driver
evaluates the statement forms the reference's scripted traces and RuleProvider emit:
``print(NodeInfo(RetrieveNode("t")))`` (the vertex chunk + "\\n", interp.cpp:68-74 /
value.cpp:88) and ``print(NodeFeature([RetrieveNode("t"), ...], "attr"))`` (value.cpp:86-125
rendering of the attribute list); anything else raises NotImplementedError.
"""
from __future__ import annotations

import ctypes as C
import json
import re
from dataclasses import dataclass, field

from . import _lib
from ._lib import check, lib
from .kvcache import PrefillReport, count_tokens, tokenize
from .templates import TemplateSet
from .workload import GraphCoTWorkload


def load_trace(path):
    """ScriptedProvider::load_jsonl (provider.cpp:36-55): {(session, agent, step): text}."""
    out = {}
    with open(path, encoding="utf-8") as f:
        for line in f:
            if not line.strip(" \t\r\n"):
                continue
            j = json.loads(line)
            out[(j["session"], j["agent"], int(j["step"]))] = j["text"]
    return out


def load_questions(path):
    """[(id, text)] of a questions JSONL ({"id", "text"}), in file order."""
    out = []
    with open(path, encoding="utf-8") as f:
        for line in f:
            if line.strip(" \t\r\n"):
                j = json.loads(line)
                out.append((j["id"], j["text"]))
    return out


# ---------------------------------------------------------------- output.cpp:36-70
class UnexpectedAgentOutput(ValueError):
    pass


def _trim(s):
    return s.strip(" \t\r\n")


def parse_classification(raw):
    """True = deterministic ("yes"), False = "no" (output.cpp:36-45)."""
    i = 0
    while i < len(raw) and raw[i] in " \t\r\n":
        i += 1
    if i == len(raw):
        raise UnexpectedAgentOutput("empty classification response")
    tok = ""
    while i < len(raw) and raw[i].isascii() and raw[i].isalpha():
        tok += raw[i].lower()
        i += 1
    if tok in ("yes", "no"):
        return tok == "yes"
    raise UnexpectedAgentOutput("classification must start with yes or no, got: " + _trim(raw))


def parse_reasoning(raw):
    """("finish", answer) or ("missing", text) (output.cpp:47-56)."""
    missing = None
    for line in raw.split("\n"):
        t = _trim(line)
        if t.startswith("Finish:"):
            return "finish", _trim(t[7:])
        if missing is None and t.startswith("Missing:"):
            missing = _trim(t[8:])
    if missing is not None:
        return "missing", missing
    raise UnexpectedAgentOutput("reasoning response has neither Finish: nor Missing: marker")


def parse_action(raw):
    """The fenced code block's body (output.cpp:58-68)."""
    o = raw.find("```")
    if o < 0:
        raise UnexpectedAgentOutput("action response has no fenced code block")
    body = raw.find("\n", o)
    if body < 0:
        raise UnexpectedAgentOutput("unterminated code fence")
    c = raw.find("```", body + 1)
    if c < 0:
        raise UnexpectedAgentOutput("unterminated code fence")
    return raw[body + 1:c]


_STR = r'"((?:[^"\\]|\\.)*)"'
_INFO = re.compile(r"^print\(NodeInfo\(RetrieveNode\(" + _STR + r"\)\)\)$")
_FEAT = re.compile(r"^print\(NodeFeature\(\[(.*)\],\s*" + _STR + r"\)\)$")
_RN = re.compile(r"RetrieveNode\(" + _STR + r"\)")


def _unescape(s):
    return json.loads('"' + s + '"')


def snippet_statements(src):
    """[(kind, [retrieve texts], attr)] of a snippet: kind "info" or "feature"."""
    out = []
    for line in src.split("\n"):
        st = line.strip()
        if not st:
            continue
        m = _INFO.match(st)
        if m:
            out.append(("info", [_unescape(m.group(1))], None))
            continue
        m = _FEAT.match(st)
        if m and _RN.sub("", m.group(1)).replace(",", "").strip() == "":
            out.append(("feature", [_unescape(x) for x in _RN.findall(m.group(1))],
                        _unescape(m.group(2))))
            continue
        raise NotImplementedError("snippet statement outside the driver's subset (the snippet "
                                  "interpreter is out of scope): " + st)
    return out


def _render_feature(value_kind):
    """Value::from_attr(...).render() (value.cpp:79-99) of one attribute, from its canonical
    rendering; a missing attribute renders as Missing."""
    if value_kind is None:
        return "Missing"
    v, kind = value_kind
    if kind == 3:  # bool: Value renders True / False (attr.hpp renders true / false)
        return "True" if v == "true" else "False"
    return v


# ---------------------------------------------------------------- the driver
@dataclass
class Record:
    """TraceRecord (orchestrator.cpp:99-114): actor, tokens_in, tokens_out, cached_tokens,
    computed_tokens (= computed + tail), outcome."""
    actor: str
    tokens_in: int
    tokens_out: int
    cached: int
    computed: int
    outcome: str

    def row(self):
        return [self.actor, self.tokens_in, self.tokens_out, self.cached, self.computed]


@dataclass
class ScriptedSession:
    sid: str
    question: str
    state: str = "C"  # C classifying, D direct action, R reasoning, A acting, done, failed
    notebook: str = ""
    rounds: int = 0
    pending_task: str = ""
    steps: dict = field(default_factory=lambda: {"classification": 0, "reasoning": 0,
                                                 "action": 0})
    records: list = field(default_factory=list)
    answer: str = ""
    error: str = ""


@dataclass
class ScriptedCall:
    session: ScriptedSession
    agent: str
    actor: str
    segments: list
    reply: str
    is_finish: bool
    report: PrefillReport = None
    first_token: int = -1
    logits: object = None
    decoded: list = field(default_factory=list)
    tokens: list = field(default_factory=list)  # the prefill's tokens (kv_prefill of segments)


class ScriptedWorkload:
    def __init__(self, engine, retriever, node_index, replies, questions, lanes=8,
                 templates=None, max_steps=10, decode=True, want_logits=False):
        self.engine = engine
        self.retriever = retriever
        self.node_index = node_index
        self.replies = replies
        self.templates = templates or TemplateSet()
        self.lanes = max(1, lanes)
        self.max_steps = max_steps
        self.decode = decode
        self.want_logits = want_logits
        self.sessions = [ScriptedSession(sid, q) for sid, q in questions]
        self.admitted = 0
        self.active = []
        self.calls = []  # every call made, in the reference's call order

    def done(self):
        return self.admitted >= len(self.sessions) and not self.active

    def _reply(self, s, agent):
        key = (s.sid, agent, s.steps[agent])
        if key not in self.replies:
            raise KeyError("no scripted entry for (%s, %s, %d)" % key)  # ProviderProtocolError
        return self.replies[key]

    def _call(self, s):
        t = self.templates
        if s.state == "C":
            return ScriptedCall(s, "classification", "C", t.render_classification(s.question),
                                self._reply(s, "classification"), False)
        if s.state == "D":  # step_direct_action: action_phase(question), then finish
            return ScriptedCall(s, "action", "A", t.render_action(s.question),
                                self._reply(s, "action"), True)
        if s.state == "R":
            reply = self._reply(s, "reasoning")
            return ScriptedCall(s, "reasoning", "R", t.render_reasoning(s.question, s.notebook),
                                reply, parse_reasoning(reply)[0] == "finish")
        return ScriptedCall(s, "action", "A", t.render_action(s.pending_task),
                            self._reply(s, "action"), False)

    def _prefill(self, calls):
        n = len(calls)
        arr, keep = GraphCoTWorkload.pack(calls)
        reps = (_lib.PrefillReportC * max(1, n))()
        first = (C.c_int32 * max(1, n))()
        lp = None
        logits = None
        if self.want_logits:
            import numpy as np
            logits = np.zeros((n, self.engine.model.cfg.vocab), dtype=np.float32)
            lp = logits.ctypes.data_as(_lib.f32p)
        check(lib().glmx_engine_prefill_segments(self.engine.h, n, arr, reps, first, lp))
        del keep
        for i, c in enumerate(calls):
            c.report = PrefillReport(reps[i].cached_tokens, reps[i].computed_tokens,
                                     reps[i].tail_tokens)
            c.first_token = first[i]
            if logits is not None:
                c.logits = logits[i]

    def _execute(self, calls):
        """Action snippets of the rotation, in lane order: RetrieveNode through K5 + the
        retrieval LRU (one batched scan), NodeInfo chunks through K1 (one batch)."""
        stmts = [snippet_statements(parse_action(c.reply)) for c in calls]
        texts = [t for ss in stmts for _, ts, _ in ss for t in ts]
        nodes = self.node_index.retrieve_nodes(texts)[0] if texts else []
        info_nodes, k = [], 0
        resolved = []
        for ss in stmts:
            rs = []
            for kind, ts, attr in ss:
                ids = nodes[k:k + len(ts)]
                k += len(ts)
                rs.append((kind, ids, attr))
                if kind == "info":
                    info_nodes.append(ids[0])
            resolved.append(rs)
        chunks = self.retriever.chunk_build(info_nodes).texts if info_nodes else []
        out, j = [], 0
        g = self.retriever.graph
        for rs in resolved:
            stdout = ""
            for kind, ids, attr in rs:
                if kind == "info":
                    stdout += chunks[j] + "\n"  # PrintStmt: raw chunk + "\n"
                    j += 1
                else:
                    stdout += "[" + ", ".join(_render_feature(g.node_attr(v, attr))
                                              for v in ids) + "]\n"
            out.append(stdout)
        return out

    def rotation(self):
        """One round-robin rotation (bench.cpp:71-83).  Returns its calls."""
        while len(self.active) < self.lanes and self.admitted < len(self.sessions):
            self.active.append(self.sessions[self.admitted])
            self.admitted += 1
        calls = []
        for s in self.active:
            if s.state == "R" and s.rounds >= self.max_steps:  # step_reasoning's step limit
                s.state, s.error = "failed", "StepLimitExceeded"
                continue
            calls.append(self._call(s))
        if calls:
            self._prefill(calls)
            for c in calls:  # Orchestrator::kv_prefill's token list (per-segment tokenize)
                c.tokens = [tok for _, text in c.segments for tok in tokenize(text)]
            steps = [max(0, count_tokens(c.reply) - 1) for c in calls]
            if self.decode and any(steps):
                cap = self.engine.max_decode
                if max(steps) > cap:
                    raise ValueError(f"a reply needs {max(steps)} decode steps > max_decode {cap}")
                dec = self.engine.decode(steps)
                for c, d in zip(calls, dec):
                    c.decoded = d
        acting = [c for c in calls if c.agent == "action"]
        stdout = dict(zip((id(c) for c in acting), self._execute(acting))) if acting else {}
        for c in calls:
            s = c.session
            s.steps[c.agent] += 1
            prompt = "".join(text for _, text in c.segments)
            r = c.report
            rec = Record(c.actor, count_tokens(prompt), count_tokens(c.reply), r.cached_tokens,
                         r.computed_tokens + r.tail_tokens, "")
            s.records.append(rec)
            if c.actor == "C":
                det = parse_classification(c.reply)
                rec.outcome = "deterministic" if det else "non-deterministic"
                s.state = "D" if det else "R"
            elif c.actor == "R":
                kind, text = parse_reasoning(c.reply)
                rec.outcome = kind
                if kind == "finish":
                    s.answer, s.state = text, "done"  # set_tier ran inside the batch
                else:
                    s.pending_task, s.state = text, "A"
            else:
                rec.outcome = "action"
                out = stdout[id(c)]
                if s.state == "D":
                    s.answer = out[:-1] if out.endswith("\n") else out  # rtrim_newline
                    s.state = "done"
                else:
                    s.notebook += out  # Notebook::append (rendered = concatenated facts)
                    s.rounds += 1
                    s.state = "R"
        self.active = [s for s in self.active if s.state not in ("done", "failed")]
        self.calls.extend(calls)
        return calls

    def run(self):
        while not self.done():
            self.rotation()
        return self.calls


def export_trace(sessions_calls):
    """ScriptedProvider trace lines (session, agent, step, text) for an iterable of
    (session id, agent, reply) in call order -- to run the reference's own orchestrator on the
    same replies (oracle ref_run_scripted)."""
    steps, out = {}, []
    for sid, agent, text in sessions_calls:
        k = (sid, agent)
        out.append({"session": sid, "agent": agent, "step": steps.get(k, 0), "text": text})
        steps[k] = steps.get(k, 0) + 1
    return out
