"""Closed-loop online planning (NEXT-4 of SURVEY §8(f)), on the public API.

At every real step:

1. the planner builds a DESPOT from the current particle belief with
   ``despot_plan`` (the host tree driver over batched GPU expansions) and
   returns a* = argmax_a l(b0, a);
2. the world -- a one-scenario belief holding the true state, drawing from
   its own random stream -- executes a*: its successor state, observation z
   and reward come from the same model step g the planner simulates;
3. the belief is updated by the particle filter the DESPOT tree implies
   (Eq. 3 with the scenarios as particles): every particle is stepped with a*
   and those whose observation equals z are kept -- exactly the update step
   (K1) of the root's child (a*, z).  The survivors are resampled (with
   replacement, weight-proportional, seeded) back to K particles; the next
   root gets fresh scenario streams (a new stream seed per step, as DESPOT
   samples new scenarios every step).

Readings: particle deprivation (no particle produced z) falls
back to the caller's prior sampler; the episode return is sum_t gamma^t r_t of
the world's rewards; an episode ends when the world's observation is TERMINAL
or after `steps` steps.  Everything runs through libdespot (no CPU model)."""
from __future__ import annotations

import numpy as np

from .despot import Model


def _terminal(model: Model, z) -> bool:
    z = np.atleast_1d(z)
    return bool(z[0] == model.slots - 1) if model.slots else bool(z[0] == 0xFFFFFFFF)


def world_step(model: Model, s, a: int, seed: int):
    """(s', z, r, terminal) of the true state s (u32 [SW]) under action a, the
    step's randomness drawn from the world's own stream `seed`."""
    node = model.belief_load(np.asarray(s, np.uint32).reshape(model.SW, 1), np.ones(1, np.float32), seed)
    R = model.expand([(node, -1, 0, 0)])
    c0, c1 = int(R["child_begin"][a]), int(R["child_begin"][a + 1])
    assert c1 - c0 == 1, "one scenario has exactly one child per action"
    z = np.array(R["child_obs"][c0]).reshape(-1).copy()
    r = float(R["act_reward"][a])
    C = model.expand([(node, a, 0, 1)])
    s2 = model.node_read(C["node"][0])["states"][:, 0].copy()
    model.node_release_many([C["node"][0], node])
    return s2, z, r, _terminal(model, z)


def belief_update(model: Model, root: int, a: int, z):
    """The particles of the root's child (a, z): (states [SW][n], weights [n]),
    or None when no particle produced z (deprivation)."""
    R = model.expand([(root, -1, 0, 0)])  # the root's child keys (the planner expanded it the same way)
    z = np.atleast_1d(np.asarray(z, np.uint32))
    c0, c1 = int(R["child_begin"][a]), int(R["child_begin"][a + 1])
    obs = np.asarray(R["child_obs"]).reshape(-1, model.OW)
    k = next((c - c0 for c in range(c0, c1) if np.array_equal(obs[c], z)), None)
    if k is None:
        return None
    C = model.expand([(root, a, k, 1)])
    rd = model.node_read(C["node"][0])
    model.node_release(C["node"][0])
    return rd["states"].copy(), rd["w"].copy()


def resample(states, w, K: int, rng: np.random.Generator):
    """K particles drawn with replacement, probability proportional to w
    (uniform weights 1/K afterwards)."""
    p = np.asarray(w, np.float64)
    idx = rng.choice(len(p), size=K, replace=True, p=p / p.sum())
    return np.ascontiguousarray(states[:, idx]), np.full(K, np.float32(1.0 / K), np.float32)


def run_episode(model: Model, prior, true_state, K: int, steps: int, config, seed: int = 0):
    """One closed-loop episode.  prior(K, seed) -> (states [SW][K], weights [K])
    samples the initial belief (and refills a deprived one); true_state is the
    world's initial state.  Returns a dict with the discounted return, the
    actions, rewards, observations, belief sizes and the per-step search
    results."""
    rng = np.random.Generator(np.random.PCG64(seed))
    states, w = prior(K, seed)
    s = np.asarray(true_state, np.uint32).copy()
    ret, disc, term = 0.0, 1.0, False
    log = dict(actions=[], rewards=[], obs=[], survivors=[], deprived=0, search=[])
    for t in range(steps):
        root = model.belief_load(states, w, (seed << 20) + 2 * t + 1)  # fresh scenario streams per step
        res = model.plan(root, config)
        a = int(res["action"])
        s, z, r, term = world_step(model, s, a, (seed << 20) + 2 * t + 2)
        ret += disc * r
        disc *= model.gamma
        log["actions"].append(a)
        log["rewards"].append(r)
        log["obs"].append(z.tolist())
        log["search"].append(res)
        if term:
            model.node_release(root)
            break
        upd = belief_update(model, root, a, z)
        model.node_release(root)
        if upd is None:
            log["deprived"] += 1
            log["survivors"].append(0)
            states, w = prior(K, (seed << 20) + 2 * t + 3)
        else:
            log["survivors"].append(int(upd[1].shape[0]))
            states, w = resample(upd[0], upd[1], K, rng)
    log.update(discounted_return=ret, steps=len(log["actions"]), terminal=term)
    return log
