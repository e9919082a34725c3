#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 "done = each oracle function
fails at least one external pin under a plausible mistake").

Copies oracle/, tests/ and workloads/ into a temporary directory, applies one
plausible mistake at a time to the copy of padsim_oracle.c, rebuilds it there
and runs the CPU oracle pin tests; a mutant must make at least one test fail.

    python tools/oracle_mutants.py > profiles/oracle_mutants_r02.txt
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = ["tests/test_oracle_mechanics.py", "tests/test_oracle_replay.py", "tests/test_oracle_controller.py",
         "tests/test_oracle_model.py", "tests/test_oracle_invariants.py"]

# name -> (passage the mistake violates, original text, mutated text)
MUTANTS = {
    "settle: decrease applied at command time": (
        "P:159-161 source-before-sink",
        "if (tgt < W[g].cmd) W[g].cmd = tgt;",
        "if (tgt < W[g].cmd) { W[g].cmd = tgt; W[g].eff = tgt; if (W[g].role == 1) W[g].dirty = 1; }"),
    "settle: raise applied at command time": (
        "P:159-161, P:291",
        "else if (tgt > W[g].cmd) W[g].raise_to = tgt;",
        "else if (tgt > W[g].cmd) { W[g].cmd = W[g].eff = tgt; }"),
    "MoveGPU: flip without the reassignment delay": (
        "P:294",
        "heap_push(&h, t + pol->reassign_s, K_FLIP, g)",
        "heap_push(&h, t, K_FLIP, g)"),
    "MoveGPU: re-route queued prompts in reverse order": (
        "S:256 (queue order)",
        "int i = ring_pop(&w->q);\n                                w->outstanding",
        "int i = w->q.buf[(w->q.head + w->q.len - 1) % w->q.cap]; w->q.len--;\n                                w->outstanding"),
    "window: exclusive lower edge": (
        "A22 window [t-W, t]",
        "if (s_ttft.stamp[k] >= lo_t && s_ttft.stamp[k] <= t)",
        "if (s_ttft.stamp[k] > lo_t && s_ttft.stamp[k] <= t)"),
    "window: TTFT stamped at completion (SPEC variant)": (
        "A22 (TTFT known at first token)",
        ["completed++; s_tpot.stamp[s_tpot.n] = (T);",
         "                    s_ttft.stamp[s_ttft.n] = t; s_ttft.val[s_ttft.n] = t - a[i]; s_ttft.n++;\n"],
        ["completed++; s_ttft.stamp[s_ttft.n] = (T); s_ttft.val[s_ttft.n] = pe[id_] - a[id_]; s_ttft.n++; "
         "s_tpot.stamp[s_tpot.n] = (T);", ""]),
    "controller: TPOT SLO never switches to phase 1": (
        "S:375",
        "ob.tpot_slo = phase2_seen ? slo->tpot[1] : slo->tpot[0];",
        "ob.tpot_slo = slo->tpot[0];"),
    "scoring: strict TTFT test": (
        "A6 (S:448, S:410)",
        "if (tt <= slo->ttft && tpot[i] <= ts) met++;\n            if (fabs(tt - slo->ttft) <= 1e-9 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;\n            if (i == 0 || comp[i] > last) last = comp[i];\n            if (o_ttft) o_ttft[i] = tt;\n            if (o_tpot) o_tpot[i] = tpot[i];\n            if (o_pe) o_pe[i] = pe[i];\n            if (o_comp) o_comp[i] = comp[i];\n            if (o_te) o_te[i] = te[i];",
        "if (tt < slo->ttft && tpot[i] <= ts) met++;\n            if (fabs(tt - slo->ttft) <= 1e-9 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;\n            if (i == 0 || comp[i] > last) last = comp[i];\n            if (o_ttft) o_ttft[i] = tt;\n            if (o_tpot) o_tpot[i] = tpot[i];\n            if (o_pe) o_pe[i] = pe[i];\n            if (o_comp) o_comp[i] = comp[i];\n            if (o_te) o_te[i] = te[i];"),
    "scoring: near band 1e-8": (
        "c.2 step 5",
        "if (fabs(tt - slo->ttft) <= 1e-9 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;\n            if (i == 0 || comp[i] > last) last = comp[i];\n            if (o_ttft) o_ttft[i] = tt;\n            if (o_tpot) o_tpot[i] = tpot[i];\n            if (o_pe) o_pe[i] = pe[i];\n            if (o_comp) o_comp[i] = comp[i];\n            if (o_te) o_te[i] = te[i];",
        "if (fabs(tt - slo->ttft) <= 1e-8 * slo->ttft || fabs(tpot[i] - ts) <= 1e-9 * ts) near++;\n            if (i == 0 || comp[i] > last) last = comp[i];\n            if (o_ttft) o_ttft[i] = tt;\n            if (o_tpot) o_tpot[i] = tpot[i];\n            if (o_pe) o_pe[i] = pe[i];\n            if (o_comp) o_comp[i] = comp[i];\n            if (o_te) o_te[i] = te[i];"),
    "routing: prefill tie to the highest id": (
        "A8",
        "if (best < 0 || W[g].outstanding < bl) { best = g; bl = W[g].outstanding; }\n                }\n                ring_push(&W[best].q, i);\n                W[best].outstanding += in_tok[i];\n                break;",
        "if (best < 0 || W[g].outstanding <= bl) { best = g; bl = W[g].outstanding; }\n                }\n                ring_push(&W[best].q, i);\n                W[best].outstanding += in_tok[i];\n                break;"),
    "decode: sequential t += L instead of t_seg + k*L": (
        "A14",
        "if (!m->ctx_growth) return t_seg + (double)k * L1;",
        "if (!m->ctx_growth) { double x = t_seg; for (int j = 0; j < k; j++) x = x + L1; return x; }"),
    "TPOT: denominator out instead of out-1": (
        "A7, P:339",
        "double tp = (t - pe[i]) / (double)(out_tok[i] - 1);",
        "double tp = (t - pe[i]) / (double)(out_tok[i]);"),
    "KV buffer: transfer latency dropped": (
        "P:285, P:339",
        "te[i] = t + or_kv_lat(m, in_tok[i]);",
        "te[i] = t;"),
    "batching: token budget exclusive": (
        "A9, S:223",
        "if (tok + in_tok[nx] > m->pb_tokens) break;\n                tok += in_tok[nx];\n                b++;\n            }\n            for (int k = 0; k < b; k++) {\n                w->batch[k]",
        "if (tok + in_tok[nx] >= m->pb_tokens) break;\n                tok += in_tok[nx];\n                b++;\n            }\n            for (int k = 0; k < b; k++) {\n                w->batch[k]"),
    "MovePower: recipients get F instead of F/|rec|": (
        "S:332",
        "long share = n_rec > 0 ? F / n_rec : 0;",
        "long share = F;"),
    "controller: cooldown >= instead of >": (
        "A20, P:231",
        "if (!((now - st->last_move) > pol->cooldown_s)) return 0;",
        "if (!((now - st->last_move) >= pol->cooldown_s)) return 0;"),
}


def main():
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    for d in ("oracle", "tests", "workloads"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
    src_path = os.path.join(tmp, "oracle", "padsim_oracle.c")
    src = open(src_path).read()
    caught = 0
    print(f"oracle mutation check: {len(MUTANTS)} mutants, pins = {' '.join(TESTS)}")
    for name, (cite, a, b) in MUTANTS.items():
        pairs = list(zip(a, b)) if isinstance(a, list) else [(a, b)]
        if any(src.count(x) < 1 for x, _ in pairs):
            print(f"MISSING-SITE  {name}")
            continue
        mutated = src
        for x, y in pairs:
            mutated = mutated.replace(x, y, 1)
        open(src_path, "w").write(mutated)
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=tmp, check=True)
        r = subprocess.run([sys.executable, "-m", "pytest", *TESTS, "-q", "-m", "not gpu and not slow", "-x",
                            "-p", "no:randomly"], cwd=tmp, capture_output=True, text=True)
        last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
        failed = r.returncode != 0
        first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
        caught += failed
        print(f"{'CAUGHT' if failed else 'MISSED'}  {name}  [{cite}]  -> {last}  {first}")
    open(src_path, "w").write(src)
    shutil.rmtree(tmp, ignore_errors=True)
    print(f"caught {caught}/{len(MUTANTS)}")
    return 0 if caught == len(MUTANTS) else 1


if __name__ == "__main__":
    sys.exit(main())
