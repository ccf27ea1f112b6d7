"""Prompt templates with tier assignment — mirror of TemplateSet / render_tiered
(templates.cpp:80-114, 157-223).  The prompt assets are the reference's shipped custom/*.prompt
files (identical to its builtin strings, templates.cpp:14-69), kept as data under prompts/."""
from __future__ import annotations

import os

HERE = os.path.dirname(os.path.abspath(__file__))
TIER_I, TIER_II, TIER_III, TIER_IV = 0, 1, 2, 3
NAMES = ("classification", "reasoning", "action", "action_repair", "baseline_thought",
         "baseline_action")


def parse(text):
    """PromptTemplate::parse (templates.cpp:118-141): [(is_slot, value)]."""
    segs, pos = [], 0
    while pos < len(text):
        o = text.find("{{", pos)
        if o < 0:
            segs.append((False, text[pos:]))
            break
        c = text.find("}}", o)
        if c < 0:
            raise ValueError("unterminated {{slot}} in template")
        if o > pos:
            segs.append((False, text[pos:o]))
        name = text[o + 2:c]
        if not name:
            raise ValueError("empty slot name in template")
        segs.append((True, name))
        pos = c + 2
    return segs


def render_tiered(segs, fills):
    """templates.cpp:80-114.  fills: {slot: (value, tier)} -> [(tier, text)]; literal text
    before the first slot is tier I, later literals take the following slot's tier, trailing
    text the last slot's tier, adjacent same-tier parts merge."""
    out = []

    def push(text, tier):
        if not text:
            return
        if out and out[-1][0] == tier:
            out[-1] = (tier, out[-1][1] + text)
        else:
            out.append((tier, text))

    pending, seen, current = "", False, TIER_I
    for is_slot, val in segs:
        if not is_slot:
            pending += val
            continue
        v, t = fills[val]
        push(pending, t if seen else TIER_I)
        pending = ""
        push(v, t)
        seen, current = True, t
    push(pending, current)
    return out


class TemplateSet:
    def __init__(self, directory=None):
        d = directory or os.path.join(HERE, "prompts")
        self.t = {}
        for n in NAMES:
            with open(os.path.join(d, n + ".prompt"), encoding="utf-8") as f:
                self.t[n] = parse(f.read())

    def render_classification(self, question):
        if not question:
            raise ValueError("question must be non-empty")
        return render_tiered(self.t["classification"], {"question": (question, TIER_IV)})

    def render_reasoning(self, question, notebook_text):
        if not question:
            raise ValueError("question must be non-empty")
        return render_tiered(self.t["reasoning"], {"notebook": (notebook_text, TIER_II),
                                                   "question": (question, TIER_IV)})

    def render_action(self, task):
        return render_tiered(self.t["action"], {"task": (task, TIER_IV)})

    def render_action_repair(self, task, failed_snippet, error):
        return render_tiered(self.t["action_repair"], {"task": (task, TIER_IV),
                                                       "failed_snippet": (failed_snippet, TIER_IV),
                                                       "error": (error, TIER_IV)})

    def render_baseline_thought(self, question, history):
        return render_tiered(self.t["baseline_thought"], {"history": (history, TIER_II),
                                                          "question": (question, TIER_IV)})

    def render_baseline_action(self, question, history):
        return render_tiered(self.t["baseline_action"], {"history": (history, TIER_II),
                                                         "question": (question, TIER_IV)})
