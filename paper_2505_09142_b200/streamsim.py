"""Closed-loop ISRTF iteration driver + stream simulator (
BASELINE.json configs[3]: Poisson arrivals, ISRTF with preemption vs FCFS, predictor on GPU).

It runs PAPER.md Algorithm 1 (alg:scheduler_flow) for W backend workers (per-node
Priority Buffers and the least-loaded balancer) with the GPU hot path in the
loop.  At every scheduling instant:
  * the due set -- new arrivals and the jobs that just ran a window (lines 10-18; jobs waiting
    in the Priority Buffer keep their cached priority, R8) -- is re-predicted by
    elis_predict_remaining straight into a device-resident in-flight table (out_slot); its
    predictor inputs are gathered on the device from the token arena (elis_arena_*: each prompt is
    uploaded once at arrival and each window's generated tokens appended, the B200 analogue of
    "the prompt is sent once ... fixed-window partial outputs");
  * elis_isrtf_select_nodes picks the next batch of every free node from its own queue
    (line 19) with the running flags of the node's previous batch (preemption,
    P:345-348) and optional aging / preemption margin (row f3);
  * the backend is modelled as windows of K = 50 tokens ending early when a member finishes
    (P:341-342), lasting TTFT (first execution) + TPOT x tokens (Sec. 2.1).
The LLM itself is out of scope: each job's response tokens are synthetic and
its true length is known to the simulator only.

Priority sources: "gpu" (the BGE + 8-FC predictor; random-init weights carry no length
signal, so this measures the mechanics and the per-iteration GPU overhead), "oracle" (true
remaining tokens: the SRTF bound, written into the table), "noisy" (SPEC's NoisyIterative:
true length + Laplace error with the MAE schedule, a stand-in for the trained predictor), "sjf"
(the true total length, a static key: shortest-job-first by the profiled length; run
without preemption) and policy FCFS.

Every GPU decision is recorded so tests can replay the run through the fp64 oracle simulator
and require identical schedules.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import binding, inputs

POLICY_ISRTF, POLICY_FCFS = binding.POLICY_ISRTF, binding.POLICY_FCFS


@dataclass
class StreamResult:
    first: np.ndarray                 # first-execution time per job (ms)
    finish: np.ndarray                # completion time per job (ms)
    arrival: np.ndarray
    iterations: int
    gpu_ms_per_iter: float            # device-side predict + select time per window (CUDA events)
    host_ms_per_iter: float           # wall clock of the whole driver step per window
    predicted_per_iter: float         # mean due-set size
    recorded: dict = field(default_factory=dict)  # (job, generated) -> fp32 priority used

    @property
    def jct(self) -> np.ndarray:
        return self.finish - self.arrival

    def summary(self) -> dict:
        return {"mean_jct_ms": float(self.jct.mean()), "mean_queue_ms": float((self.first - self.arrival).mean()),
                "iterations": self.iterations, "gpu_ms_per_iter": self.gpu_ms_per_iter,
                "host_ms_per_iter": self.host_ms_per_iter, "due_per_iter": self.predicted_per_iter}


def build_sequence(prompt: np.ndarray, response: np.ndarray, generated: int, max_len: int = 512) -> np.ndarray:
    """'the prompt attached with the answer': [CLS] prompt [SEP] + the response so far.
    Longer than max_len: keep the most recent <= 254 response tokens and the head of the prompt
    (R7)."""
    resp = response[:generated]
    if prompt.size + resp.size <= max_len:
        return np.concatenate([prompt, resp]).astype(np.int32)
    keep_resp = min(resp.size, 254)
    head = prompt[:max_len - keep_resp]
    return np.concatenate([head, resp[resp.size - keep_resp:]]).astype(np.int32)


def seq_len(prompt_len: int, generated: int, max_len: int = 512) -> int:
    """Length of build_sequence's output (R7)."""
    if prompt_len + generated <= max_len:
        return prompt_len + generated
    keep = min(generated, 254)
    return min(prompt_len, max_len - keep) + keep


class StreamSim:
    """Algorithm 1 over `workers` backend nodes with per-node Priority Buffers:
    arrivals go to the least-loaded node (elis_assign_nodes), every free node forms its batch
    from its own queue in one elis_isrtf_select_nodes launch, with optional starvation control
    (aging / preemption margin, R17).  Event order at an instant t (R18): windows
    ending at t complete, arrivals up to t are admitted, free nodes form batches."""

    def __init__(self, predictor: binding.Predictor | None, policy: int = POLICY_ISRTF, cap: int = 4,
                 window: int = inputs.WINDOW_K, ttft_ms: float = 0.0, tpot_ms: float = 1.0,
                 allow_preempt: bool = True, priority: str = "gpu", seed: int = 0, workers: int = 1,
                 boost_after: int = 1, boost_amount: float = 0.0, preempt_margin: float = 0.0,
                 arena: bool = True, graph: bool = True):
        if priority == "gpu" and predictor is None and policy == POLICY_ISRTF:
            raise ValueError("priority='gpu' needs a predictor")
        self.P = predictor
        self.policy, self.cap, self.K = policy, cap, window
        self.ttft, self.tpot, self.allow = ttft_ms, tpot_ms, allow_preempt
        self.priority, self.seed, self.W = priority, seed, workers
        self.boost_after, self.boost_amount, self.margin = boost_after, boost_amount, preempt_margin
        self.use_arena = arena
        self.use_graph = graph and arena

    def run(self, prompts, totals, arrivals_ms, select_predictor: binding.Predictor | None = None) -> StreamResult:
        import torch
        P = self.P if self.P is not None else select_predictor
        if P is None:
            raise ValueError("a predictor (for the device select) is required")
        nj, W, cap = len(prompts), self.W, self.cap
        order = np.argsort(arrivals_ms, kind="stable")
        assert (order == np.arange(nj)).all(), "jobs must be sorted by arrival (id = arrival rank)"
        responses = [inputs.response_tokens(j, int(totals[j]), self.seed) for j in range(nj)]
        gen = np.full(nj, -1, np.int32)            # -1: not arrived or finished (ineligible slot)
        node_of = np.full(nj, -1, np.int32)
        waited = np.zeros(nj, np.int32)
        first = np.full(nj, np.nan)
        finish = np.full(nj, np.nan)
        running = np.zeros(nj, np.uint8)
        started = np.zeros(nj, bool)
        free_at = [None] * W
        batch_of: list[list[int]] = [[] for _ in range(W)]
        tokens_of = [0] * W
        dev = torch.device("cuda")
        st = torch.cuda.Stream()             # a side stream: CUDA graphs cannot be captured on the default one
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            return self._loop(P, torch, dev, st, nj, W, cap, prompts, totals, arrivals_ms, responses, gen, node_of,
                              waited, first, finish, running, started, free_at, batch_of, tokens_of)

    def _loop(self, P, torch, dev, st, nj, W, cap, prompts, totals, arrivals_ms, responses, gen, node_of, waited,
              first, finish, running, started, free_at, batch_of, tokens_of):
        d_table = torch.zeros(nj, device=dev)
        d_gen = torch.empty(nj, dtype=torch.int32, device=dev)
        d_run = torch.empty(nj, dtype=torch.uint8, device=dev)
        d_node = torch.empty(nj, dtype=torch.int32, device=dev)
        d_wait = torch.empty(nj, dtype=torch.int32, device=dev)
        d_ready = torch.empty(W, dtype=torch.uint8, device=dev)
        d_load = torch.zeros(W, dtype=torch.int32, device=dev)
        d_newnode = torch.empty(max(nj, 1), dtype=torch.int32, device=dev)
        d_order = torch.arange(nj, dtype=torch.int32, device=dev).to(torch.int32)
        d_ids = torch.empty(W * cap, dtype=torch.int32, device=dev)
        d_cnt = torch.empty(W, dtype=torch.int32, device=dev)
        h_ids = torch.empty(W * cap, dtype=torch.int32).pin_memory()
        h_cnt = torch.empty(W, dtype=torch.int32).pin_memory()
        aging = self.boost_amount != 0.0
        gpu_pred = self.priority == "gpu" and self.policy == POLICY_ISRTF
        arena = binding.Arena(nj) if (gpu_pred and self.use_arena) else None
        plen = np.array([len(q) for q in prompts], np.int64)
        d_seq = torch.empty(max(nj, 1) * 512 if arena is not None else 1, dtype=torch.int32, device=dev)
        d_seqlen = torch.empty(max(nj, 1), dtype=torch.int32, device=dev)
        app_slots, app_toks, app_cnts = [], [], []   # this iteration's generated tokens (arena appends)
        d_slots = torch.zeros(max(nj, 1), dtype=torch.int32, device=dev)
        d_dims = torch.zeros(2, dtype=torch.int32, device=dev)
        graph, eager_done = None, False

        def predict_select():
            # shape-agnostic predict (n, T from d_dims, written by the arena gather) + the select:
            # one CUDA graph replayed every iteration whatever the due set's size
            P.predict_remaining_dev(d_seq, d_seqlen, d_dims, d_table, out_slot=d_slots, stream=st)
            select()

        def select():
            P.isrtf_select_nodes(d_table, d_gen, d_node, W, cap, d_ids, d_cnt, node_ready=d_ready,
                                 policy=self.policy, allow_preempt=self.allow, order=d_order, running=d_run,
                                 stream=st, windows_waited=d_wait if aging else None, boost_after=self.boost_after,
                                 boost_amount=self.boost_amount, preempt_margin=self.margin)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        recorded = {}
        nxt = 0                                     # next job to arrive
        due: list[int] = []
        iters, selects, gpu_ms, host_ms, due_total = 0, 0, 0.0, 0.0, 0
        done = 0
        while done < nj:
            ends = [f for f in free_at if f is not None]
            t = min(min(ends) if ends else np.inf, float(arrivals_ms[nxt]) if nxt < nj else np.inf)
            h0 = time.perf_counter()
            # (a) windows ending at t
            for w in range(W):
                if free_at[w] is not None and free_at[w] <= t:
                    running[node_of == w] = 0
                    for j in batch_of[w]:
                        if arena is not None and gen[j] + tokens_of[w] < totals[j]:
                            app_slots.append(j)
                            app_toks.append(responses[j][gen[j]:gen[j] + tokens_of[w]])
                            app_cnts.append(tokens_of[w])
                        gen[j] += tokens_of[w]
                        if gen[j] >= totals[j]:
                            finish[j] = free_at[w]
                            gen[j] = -1
                            done += 1
                            d_load[w] -= 1
                        else:
                            running[j] = 1
                            due.append(j)
                    free_at[w], batch_of[w] = None, []
            # (b) arrivals: least-loaded node on the device
            n_new = 0
            while nxt + n_new < nj and arrivals_ms[nxt + n_new] <= t:
                n_new += 1
            ev0.record(st)
            if n_new and arena is not None:   # each prompt crosses PCIe once
                arena.set_prompts(torch.arange(nxt, nxt + n_new, dtype=torch.int32).to(dev, non_blocking=True),
                                  torch.from_numpy(np.concatenate(prompts[nxt:nxt + n_new]).astype(np.int32)).to(
                                      dev, non_blocking=True),
                                  torch.from_numpy(plen[nxt:nxt + n_new].astype(np.int32)).to(dev, non_blocking=True),
                                  stream=st)
            if app_slots:                      # ... and each window's generated tokens once
                arena.append(torch.from_numpy(np.array(app_slots, np.int32)).to(dev, non_blocking=True),
                             torch.from_numpy(np.concatenate(app_toks).astype(np.int32)).to(dev, non_blocking=True),
                             torch.from_numpy(np.array(app_cnts, np.int32)).to(dev, non_blocking=True), stream=st)
                app_slots, app_toks, app_cnts = [], [], []
            if n_new:
                P.assign_nodes(d_load, n_new, d_newnode, stream=st)
                node_of[nxt:nxt + n_new] = d_newnode[:n_new].cpu().numpy()
                gen[nxt:nxt + n_new] = 0
                waited[nxt:nxt + n_new] = 0
                due.extend(range(nxt, nxt + n_new))
                nxt += n_new
            # (c) free nodes with work form their batches (one segmented select)
            ready = np.array([free_at[w] is None for w in range(W)], np.uint8)
            has_work = np.zeros(W, bool)
            live = gen >= 0
            has_work[np.unique(node_of[live])] = True
            for w in range(W):
                if ready[w] and not has_work[w]:
                    running[node_of == w] = 0
            if not (ready.astype(bool) & has_work).any():
                ev1.record(st)
                continue
            if due and self.policy == POLICY_ISRTF:
                if self.priority == "gpu" and arena is not None and self.use_graph:
                    # predictor inputs gathered on the device (d_dims = {n, total}); predict + select
                    # below, from the captured graph
                    d_slots[:len(due)].copy_(torch.from_numpy(np.array(due, np.int32)), non_blocking=True)
                    arena.gather(d_slots[:len(due)], 512, d_seq, d_seqlen, out_dims=d_dims, stream=st)
                elif self.priority == "gpu" and arena is not None:
                    # predictor inputs gathered on the device; the host knows their total from the
                    # prompt lengths and generated counts (the same R7 rule)
                    slots = torch.from_numpy(np.array(due, np.int32)).to(dev, non_blocking=True)
                    total = int(sum(seq_len(int(plen[j]), int(gen[j])) for j in due))
                    arena.gather(slots, 512, d_seq, d_seqlen[:len(due)], stream=st)
                    P.predict_remaining(d_seq, d_seqlen[:len(due)], total, d_table, out_slot=slots, stream=st)
                elif self.priority == "gpu":
                    seqs = [build_sequence(prompts[j], responses[j], int(gen[j])) for j in due]
                    lens = np.array([q.size for q in seqs], np.int32)
                    toks = torch.from_numpy(np.concatenate(seqs)).to(dev, non_blocking=True)
                    slots = torch.from_numpy(np.array(due, np.int32)).to(dev, non_blocking=True)
                    P.predict_remaining(toks, torch.from_numpy(lens).to(dev, non_blocking=True), int(lens.sum()),
                                        d_table, out_slot=slots, stream=st)
                else:  # "oracle": true remaining tokens (SRTF bound); "noisy": SPEC NoisyIterative;
                    # "sjf": the job's true total length, fixed for its lifetime (SJF by the
                    # profiled length; R16 reading of SV)
                    if self.priority == "sjf":
                        rem = totals[due].astype(np.float32)
                    elif self.priority == "noisy":
                        rem = np.array([inputs.noisy_remaining(j, int(totals[j]), int(gen[j]), self.seed)
                                        for j in due], np.float32)
                    else:
                        rem = (totals[due] - gen[due]).astype(np.float32)
                    d_table[torch.from_numpy(np.array(due, np.int64)).to(dev)] = torch.from_numpy(rem).to(dev)
            d_gen.copy_(torch.from_numpy(gen), non_blocking=True)
            d_run.copy_(torch.from_numpy(running), non_blocking=True)
            d_node.copy_(torch.from_numpy(node_of), non_blocking=True)
            d_ready.copy_(torch.from_numpy(ready), non_blocking=True)
            if aging:
                d_wait.copy_(torch.from_numpy(waited), non_blocking=True)
            if self.use_graph and gpu_pred:
                if not due:
                    d_dims.zero_()             # nothing to re-predict: the graph's predict is a no-op
                if graph is None and eager_done:
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph, stream=st):
                        predict_select()
                if graph is not None:
                    graph.replay()
                else:                          # first iteration: eager (sets the launch attributes)
                    predict_select()
                    eager_done = True
            else:
                select()
            h_ids.copy_(d_ids, non_blocking=True)
            h_cnt.copy_(d_cnt, non_blocking=True)
            ev1.record(st)
            st.synchronize()
            gpu_ms += ev0.elapsed_time(ev1)
            selects += 1
            if due and self.policy == POLICY_ISRTF:
                vals = d_table[torch.from_numpy(np.array(due, np.int64)).to(dev)].cpu().numpy()
                for j, v in zip(due, vals):
                    recorded[(int(j), int(gen[j]))] = float(v)
            due_total += len(due)
            due = []
            ids_all, cnts = h_ids.numpy().reshape(W, cap), h_cnt.numpy()
            for w in range(W):
                if not ready[w] or not has_work[w]:
                    continue
                batch = [int(x) for x in ids_all[w, :int(cnts[w])]]
                assert batch, "select returned an empty batch for a node with eligible jobs"
                mine = live & (node_of == w)
                waited[mine] += 1
                waited[batch] = 0
                tok = min(self.K, min(int(totals[j] - gen[j]) for j in batch))
                dur = (self.ttft if any(not started[j] for j in batch) else 0.0) + self.tpot * tok
                for j in batch:
                    if not started[j]:
                        started[j] = True
                        first[j] = t
                batch_of[w], tokens_of[w], free_at[w] = batch, tok, t + dur
                iters += 1
            host_ms += (time.perf_counter() - h0) * 1e3
        if arena is not None:
            assert arena.sync_status(st) == 0, binding.lib().elis_last_error()
            arena.close()
        return StreamResult(first, finish, np.asarray(arrivals_ms, float), iters, gpu_ms / max(selects, 1),
                            host_ms / max(selects, 1), due_total / max(selects, 1), recorded)
