// oracle/oracle.cpp -- plain CPU oracle for the GWTF routing min-cost-flow hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Deliberately simple: explicit
// residual-arc enumeration, std::priority_queue Dijkstra, sequential loops that
// follow DESIGN.md section 2 phase by phase.  No blocking, fusion or reordering
// beyond what the definitions state.  Shares no code with the CUDA path.
#include "oracle.h"

#include <chrono>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <queue>
#include <thread>
#include <tuple>
#include <vector>

namespace {

constexpr int32_t ABSENT = INT32_MAX;
constexpr int64_t INF = INT64_MAX;
constexpr int64_t CAP_INF = INT64_MAX;

// ---------------------------------------------------------------------------
// Instance (SURVEY C1; PAPER.md:137 capacities, :164-171 costs)
// ---------------------------------------------------------------------------
struct Inst {
  int S = 0, n = 0, MC = 0;
  int64_t M = 0;
  std::vector<int32_t> cap;
  std::vector<uint8_t> alive;
  std::vector<int32_t> src, snk, link;

  explicit Inst(const orc_instance* I) {
    S = I->S; n = I->n; MC = I->max_cap; M = I->M;
    cap.assign(I->cap, I->cap + (size_t)S * n);
    alive.assign((size_t)S * n, 1);
    if (I->alive) alive.assign(I->alive, I->alive + (size_t)S * n);
    src.assign(I->src, I->src + n);
    snk.assign(I->snk, I->snk + n);
    if (S > 1) link.assign(I->link, I->link + (size_t)(S - 1) * n * n);
  }
  Inst() = default;
  // effective capacity: a crashed relay holds nothing
  int32_t capE(int s, int i) const { return alive[(size_t)s * n + i] ? cap[(size_t)s * n + i] : 0; }
  // d(u in stage s -> v in stage s+1)
  int32_t C(int s, int v, int u) const { return link[((size_t)s * n + v) * n + u]; }
  int32_t& Cref(int s, int v, int u) { return link[((size_t)s * n + v) * n + u]; }
};

// ---------------------------------------------------------------------------
// Eq. 1, doubled to integer half-units
// ---------------------------------------------------------------------------
int64_t eq1_d2(int32_t ci, int32_t cj, int32_t lij, int32_t lji, int32_t bij, int32_t bji, int64_t size) {
  // 2*d = (c_i + c_j) + (lam_ij + lam_ji) + 2 * (2*size/(beta_ij+beta_ji)), transfer term floored
  return (int64_t)ci + cj + lij + lji + (4 * size) / ((int64_t)bij + bji);
}

// ---------------------------------------------------------------------------
// Successive shortest paths
// ---------------------------------------------------------------------------
struct Flow {
  std::vector<int32_t> g, src_f, snk_f, arc;  // arc[s][v][u] = f(u in s -> v in s+1)
  int64_t F = 0, cost = 0;
  int32_t A = 0;
  Flow(const Inst& I) {
    g.assign((size_t)I.S * I.n, 0);
    src_f.assign(I.n, 0);
    snk_f.assign(I.n, 0);
    arc.assign(I.S > 1 ? (size_t)(I.S - 1) * I.n * I.n : 0, 0);
  }
  int32_t& f(const Inst& I, int s, int u, int v) { return arc[((size_t)s * I.n + v) * I.n + u]; }
  int32_t fc(const Inst& I, int s, int u, int v) const { return arc[((size_t)s * I.n + v) * I.n + u]; }
};

struct Arc { int other; int64_t cost; int64_t rescap; };

// Node numbering: layer l in [0, 2S+1] (s* = 0, in_s = 2s+1, out_s = 2s+2, t* = 2S+1),
// id = l*n + position.  This is also the canonical (layer, position) order of C2.
struct Graph {
  const Inst& I;
  const Flow& f;
  int S, n;
  Graph(const Inst& I_, const Flow& f_) : I(I_), f(f_), S(I_.S), n(I_.n) {}
  int N() const { return (2 * S + 2) * n; }
  int sstar() const { return 0; }
  int tstar() const { return (2 * S + 1) * n; }
  int in(int s, int i) const { return (2 * s + 1) * n + i; }
  int out(int s, int i) const { return (2 * s + 2) * n + i; }

  // Residual arcs leaving x (arc weight (cost, 1 hop)).
  void out_arcs(int x, std::vector<Arc>& a) const {
    a.clear();
    const int l = x / n, p = x % n;
    if (x == sstar()) {
      for (int i = 0; i < n; ++i)
        if (I.src[i] != ABSENT) a.push_back({in(0, i), I.src[i], CAP_INF});
    } else if (x == tstar()) {
      for (int i = 0; i < n; ++i)
        if (f.snk_f[i] > 0) a.push_back({out(S - 1, i), -(int64_t)I.snk[i], f.snk_f[i]});
    } else if (l == 0 || l == 2 * S + 1) {
      // unused positions of the s*/t* layers
    } else if (l % 2 == 1) {  // in_{s,p}
      const int s = (l - 1) / 2, i = p;
      const int32_t g = f.g[(size_t)s * n + i];
      if (g < I.capE(s, i)) a.push_back({out(s, i), 0, (int64_t)I.capE(s, i) - g});
      if (s == 0) {
        if (f.src_f[i] > 0) a.push_back({sstar(), -(int64_t)I.src[i], f.src_f[i]});
      } else {
        for (int u = 0; u < n; ++u)
          if (f.fc(I, s - 1, u, i) > 0) a.push_back({out(s - 1, u), -(int64_t)I.C(s - 1, i, u), f.fc(I, s - 1, u, i)});
      }
    } else {  // out_{s,p}
      const int s = l / 2 - 1, i = p;
      const int32_t g = f.g[(size_t)s * n + i];
      if (g > 0) a.push_back({in(s, i), 0, g});
      if (s < S - 1) {
        for (int v = 0; v < n; ++v)
          if (I.C(s, v, i) != ABSENT) a.push_back({in(s + 1, v), I.C(s, v, i), CAP_INF});
      } else {
        if (I.snk[i] != ABSENT) a.push_back({tstar(), I.snk[i], CAP_INF});
      }
    }
  }

  // Residual arcs entering x (written separately from out_arcs; a test checks the two agree).
  void in_arcs(int x, std::vector<Arc>& a) const {
    a.clear();
    const int l = x / n, p = x % n;
    if (x == sstar()) {
      for (int i = 0; i < n; ++i)
        if (f.src_f[i] > 0) a.push_back({in(0, i), -(int64_t)I.src[i], f.src_f[i]});
    } else if (x == tstar()) {
      for (int i = 0; i < n; ++i)
        if (I.snk[i] != ABSENT) a.push_back({out(S - 1, i), I.snk[i], CAP_INF});
    } else if (l == 0 || l == 2 * S + 1) {
    } else if (l % 2 == 1) {  // in_{s,p}
      const int s = (l - 1) / 2, i = p;
      if (s == 0) {
        if (I.src[i] != ABSENT) a.push_back({sstar(), I.src[i], CAP_INF});
      } else {
        for (int u = 0; u < n; ++u)
          if (I.C(s - 1, i, u) != ABSENT) a.push_back({out(s - 1, u), I.C(s - 1, i, u), CAP_INF});
      }
      const int32_t g = f.g[(size_t)s * n + i];
      if (g > 0) a.push_back({out(s, i), 0, g});
    } else {  // out_{s,p}
      const int s = l / 2 - 1, i = p;
      const int32_t g = f.g[(size_t)s * n + i];
      if (g < I.capE(s, i)) a.push_back({in(s, i), 0, (int64_t)I.capE(s, i) - g});
      if (s < S - 1) {
        for (int v = 0; v < n; ++v)
          if (f.fc(I, s, i, v) > 0) a.push_back({in(s + 1, v), -(int64_t)I.C(s, v, i), f.fc(I, s, i, v)});
      } else {
        if (f.snk_f[i] > 0) a.push_back({tstar(), -(int64_t)I.snk[i], f.snk_f[i]});
      }
    }
  }
};

struct Key {
  int64_t c, h;  // (cost, hops), compared lexicographically
  bool operator<(const Key& o) const { return c < o.c || (c == o.c && h < o.h); }
  bool operator==(const Key& o) const { return c == o.c && h == o.h; }
};
const Key KINF{INF, INF};

// Lexicographic shortest (cost, hops) keys from s* in the residual graph, by
// Dijkstra on reduced costs with potentials pi (previous keys' cost part).
int dijkstra(const Graph& G, std::vector<int64_t>& pi, std::vector<Key>& key) {
  const int N = G.N();
  std::vector<Key> red(N, KINF);
  std::vector<char> done(N, 0);
  using E = std::tuple<int64_t, int64_t, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
  red[G.sstar()] = {0, 0};
  pq.push({0, 0, G.sstar()});
  std::vector<Arc> arcs;
  while (!pq.empty()) {
    auto [rc, rh, u] = pq.top();
    pq.pop();
    if (done[u]) continue;
    done[u] = 1;
    G.out_arcs(u, arcs);
    for (const Arc& a : arcs) {
      const int v = a.other;
      if (pi[v] == INF) return -1;  // an unreachable node can never become reachable (C2)
      const int64_t w = a.cost + pi[u] - pi[v];
      if (w < 0) return -2;  // reduced costs of residual arcs are non-negative (SSP invariant)
      const Key cand{rc + w, rh + 1};
      if (cand < red[v]) {
        red[v] = cand;
        pq.push({cand.c, cand.h, v});
      }
    }
  }
  key.assign(N, KINF);
  for (int x = 0; x < N; ++x)
    if (red[x].c != INF) key[x] = {red[x].c + pi[x] - pi[G.sstar()], red[x].h};
  return 0;
}

int ssp(const Inst& I, Flow& fl, std::vector<int64_t>* curve) {
  Graph G(I, fl);
  const int N = G.N();
  std::vector<int64_t> pi(N, 0);  // zero flow, non-negative costs: pi = 0 is feasible
  std::vector<Key> key;
  std::vector<Arc> arcs;
  if (curve) curve->assign(1, 0);
  while (fl.F < I.M) {
    int rc = dijkstra(G, pi, key);
    if (rc) return rc;
    if (key[G.tstar()].c == INF) break;  // t* unreachable: F is maximum
    // canonical predecessor: lowest (layer, position) tight in-arc (C2)
    std::vector<int> path{G.tstar()};
    int x = G.tstar();
    while (x != G.sstar()) {
      G.in_arcs(x, arcs);
      int best = -1;
      for (const Arc& a : arcs) {
        const Key& ku = key[a.other];
        if (ku.c == INF) continue;
        if (Key{ku.c + a.cost, ku.h + 1} == key[x] && (best < 0 || a.other < best)) best = a.other;
      }
      if (best < 0) return -3;
      x = best;
      path.push_back(x);
      if ((int)path.size() > N + 1) return -4;  // the predecessor graph must be acyclic
    }
    std::reverse(path.begin(), path.end());
    // bottleneck delta = min(M - F, residual capacities along the path)
    int64_t delta = I.M - fl.F, pcost = 0;
    for (size_t e = 0; e + 1 < path.size(); ++e) {
      G.out_arcs(path[e], arcs);
      const Arc* hit = nullptr;
      for (const Arc& a : arcs) if (a.other == path[e + 1]) hit = &a;
      if (!hit) return -5;
      delta = std::min(delta, hit->rescap);
      pcost += hit->cost;
    }
    if (pcost != key[G.tstar()].c || delta <= 0) return -6;
    // augment
    const int n = I.n;
    for (size_t e = 0; e + 1 < path.size(); ++e) {
      const int u = path[e], v = path[e + 1];
      const int lu = u / n, lv = v / n, pu = u % n, pv = v % n;
      if (u == G.sstar()) fl.src_f[pv] += (int32_t)delta;                       // s* -> in_0
      else if (v == G.tstar()) fl.snk_f[pu] += (int32_t)delta;                  // out_{S-1} -> t*
      else if (lu % 2 == 1 && lv == lu + 1) fl.g[(size_t)((lu - 1) / 2) * n + pu] += (int32_t)delta;  // in -> out
      else if (lu % 2 == 0 && lv == lu - 1) fl.g[(size_t)(lu / 2 - 1) * n + pu] -= (int32_t)delta;    // out -> in (reverse)
      else if (lu % 2 == 0 && lv == lu + 1) fl.f(I, lu / 2 - 1, pu, pv) += (int32_t)delta;           // out_s -> in_{s+1}
      else if (lu % 2 == 1 && lv == lu - 1) fl.f(I, lv / 2 - 1, pv, pu) -= (int32_t)delta;  // in_{s+1} -> out_s
      else return -7;
    }
    fl.F += delta;
    fl.cost += delta * key[G.tstar()].c;
    fl.A += 1;
    if (curve) curve->push_back(fl.cost);
    // potentials for the next Dijkstra: this round's cost labels; unreached nodes stay INF
    for (int y = 0; y < N; ++y) pi[y] = key[y].c;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Network simplex cross-check (SURVEY C3 i): node-split graph, supply M at s*,
// demand M at t*, bypass s*->t* with cost BIG > any simple residual path cost.
// Strongly feasible spanning trees (Cunningham) for anti-cycling; Dantzig
// entering rule; potentials recomputed by a tree walk after every pivot.
// ---------------------------------------------------------------------------
struct NSArc { int u, v; int64_t cap, cost, x; };

int network_simplex(const Inst& I, int64_t* Fout, int64_t* cost_out) {
  const int S = I.S, n = I.n;
  auto in = [&](int s, int i) { return 2 + (s * n + i) * 2; };
  auto out = [&](int s, int i) { return 3 + (s * n + i) * 2; };
  const int sstar = 0, tstar = 1, Nreal = 2 + 2 * S * n, root = Nreal, N = Nreal + 1;
  int64_t maxc = 0;
  auto upd = [&](int32_t c) { if (c != ABSENT) maxc = std::max<int64_t>(maxc, c); };
  for (int32_t c : I.src) upd(c);
  for (int32_t c : I.snk) upd(c);
  for (int32_t c : I.link) upd(c);
  const int64_t BIG = (int64_t)(2 * S * n + 2) * maxc + 1;
  const int64_t ART = 4 * BIG + 4;
  const int64_t UINF = std::max<int64_t>(I.M, 1) * 4 + 4;
  std::vector<NSArc> A;
  for (int i = 0; i < n; ++i)
    if (I.src[i] != ABSENT) A.push_back({sstar, in(0, i), UINF, I.src[i], 0});
  for (int s = 0; s < S; ++s)
    for (int i = 0; i < n; ++i) A.push_back({in(s, i), out(s, i), I.capE(s, i), 0, 0});
  for (int s = 0; s + 1 < S; ++s)
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u)
        if (I.C(s, v, u) != ABSENT) A.push_back({out(s, u), in(s + 1, v), UINF, I.C(s, v, u), 0});
  for (int i = 0; i < n; ++i)
    if (I.snk[i] != ABSENT) A.push_back({out(S - 1, i), tstar, UINF, I.snk[i], 0});
  const int bypass = (int)A.size();
  A.push_back({sstar, tstar, UINF, BIG, 0});
  const int nreal_arcs = (int)A.size();
  std::vector<int64_t> b(N, 0);
  b[sstar] = I.M;
  b[tstar] = -I.M;
  // strongly feasible initial tree: zero-flow artificial arcs point away from the root
  std::vector<int> parent(N, -1), parc(N, -1);
  for (int v = 0; v < Nreal; ++v) {
    if (b[v] > 0) A.push_back({v, root, CAP_INF, ART, b[v]});
    else A.push_back({root, v, CAP_INF, ART, -b[v]});
    parent[v] = root;
    parc[v] = (int)A.size() - 1;
  }
  std::vector<char> intree(A.size(), 0);
  for (int v = 0; v < Nreal; ++v) intree[parc[v]] = 1;
  std::vector<int64_t> pi(N, 0);
  std::vector<int> depth(N, 0);
  std::vector<std::vector<int>> ch(N);
  auto rebuild = [&]() {
    for (auto& c : ch) c.clear();
    for (int v = 0; v < N; ++v) if (v != root) ch[parent[v]].push_back(v);
    std::vector<int> st{root};
    pi[root] = 0; depth[root] = 0;
    while (!st.empty()) {
      int p = st.back(); st.pop_back();
      for (int v : ch[p]) {
        const NSArc& a = A[parc[v]];
        // reduced cost c - pi_u + pi_v = 0 on tree arcs
        pi[v] = (a.u == p) ? pi[p] - a.cost : pi[p] + a.cost;
        depth[v] = depth[p] + 1;
        st.push_back(v);
      }
    }
  };
  rebuild();
  for (long iter = 0; iter < 100000000L; ++iter) {
    int ent = -1;
    bool up = true;  // true: flow increases on the entering arc (at lower bound, rc < 0)
    int64_t best = 0;
    for (int e = 0; e < (int)A.size(); ++e) {
      if (intree[e]) continue;
      const NSArc& a = A[e];
      const int64_t rc = a.cost - pi[a.u] + pi[a.v];
      // non-tree arcs sit at a bound; an arc with cap 0 sits at both and is never eligible
      if (rc < 0 && a.x < a.cap && -rc > best) { best = -rc; ent = e; up = true; }
      if (rc > 0 && a.x > 0 && rc > best) { best = rc; ent = e; up = false; }
    }
    if (ent < 0) break;
    // push direction across the entering arc: k -> l
    const int k = up ? A[ent].u : A[ent].v, l = up ? A[ent].v : A[ent].u;
    // apex
    int a1 = k, a2 = l;
    while (a1 != a2) {
      if (depth[a1] >= depth[a2]) a1 = parent[a1]; else a2 = parent[a2];
    }
    const int apex = a1;
    // traversal in orientation starting at apex: apex -> ... -> k, (k,l), l -> ... -> apex
    struct Step { int arc; bool fwd; int child; };
    std::vector<Step> p1, p2;
    for (int v = k; v != apex; v = parent[v]) {  // tree arc between v and parent; traversed parent -> v
      const NSArc& a = A[parc[v]];
      p1.push_back({parc[v], a.u == parent[v], v});
    }
    std::reverse(p1.begin(), p1.end());
    for (int v = l; v != apex; v = parent[v]) {  // traversed v -> parent
      const NSArc& a = A[parc[v]];
      p2.push_back({parc[v], a.u == v, v});
    }
    std::vector<Step> cyc = p1;
    cyc.push_back({ent, up, -1});
    cyc.insert(cyc.end(), p2.begin(), p2.end());
    int64_t delta = CAP_INF;
    int leave = -1;
    for (int t = 0; t < (int)cyc.size(); ++t) {
      const NSArc& a = A[cyc[t].arc];
      const int64_t r = cyc[t].fwd ? (a.cap == CAP_INF ? CAP_INF : a.cap - a.x) : a.x;
      if (r <= delta) { delta = r; leave = t; }  // last blocking arc in orientation order
    }
    if (delta == CAP_INF) return -10;  // unbounded: impossible with a bypass arc
    for (const Step& st : cyc) A[st.arc].x += st.fwd ? delta : -delta;
    const Step L = cyc[leave];
    if (L.arc == ent) continue;
    // re-hang the subtree cut off by the leaving arc on the entering arc
    intree[L.arc] = 0;
    intree[ent] = 1;
    const bool on_p1 = leave < (int)p1.size();
    int v = on_p1 ? k : l, newp = on_p1 ? l : k, newarc = ent;
    const int stop = L.child;
    while (true) {
      const int oldp = parent[v], oldarc = parc[v];
      parent[v] = newp;
      parc[v] = newarc;
      if (v == stop) break;
      newp = v;
      newarc = oldarc;
      v = oldp;
    }
    rebuild();
  }
  for (int e = nreal_arcs; e < (int)A.size(); ++e)
    if (A[e].x != 0) return -11;
  int64_t total = 0;
  for (int e = 0; e < nreal_arcs; ++e) total += A[e].x * A[e].cost;
  const int64_t xb = A[bypass].x;
  *Fout = I.M - xb;
  *cost_out = total - BIG * xb;
  return 0;
}

// ---------------------------------------------------------------------------
// Certificates (SURVEY C3 iv)
// ---------------------------------------------------------------------------
int certify(const Inst& I, const Flow& fl, int64_t F, int64_t cost) {
  const int S = I.S, n = I.n;
  int64_t fsrc = 0, fsnk = 0, c = 0;
  for (int i = 0; i < n; ++i) {
    if (fl.src_f[i] < 0 || fl.snk_f[i] < 0) return 1;
    if (fl.src_f[i] > 0 && I.src[i] == ABSENT) return 1;
    if (fl.snk_f[i] > 0 && I.snk[i] == ABSENT) return 1;
    fsrc += fl.src_f[i];
    fsnk += fl.snk_f[i];
    c += (int64_t)fl.src_f[i] * (fl.src_f[i] ? I.src[i] : 0) + (int64_t)fl.snk_f[i] * (fl.snk_f[i] ? I.snk[i] : 0);
  }
  for (int s = 0; s + 1 < S; ++s)
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u) {
        const int32_t x = fl.fc(I, s, u, v);
        if (x < 0 || (x > 0 && I.C(s, v, u) == ABSENT)) return 2;
        if (x) c += (int64_t)x * I.C(s, v, u);
      }
  for (int s = 0; s < S; ++s)
    for (int i = 0; i < n; ++i) {
      const int32_t g = fl.g[(size_t)s * n + i];
      if (g < 0 || g > I.capE(s, i)) return 3;
      int64_t inflow = 0, outflow = 0;
      if (s == 0) inflow = fl.src_f[i];
      else for (int u = 0; u < n; ++u) inflow += fl.fc(I, s - 1, u, i);
      if (s == S - 1) outflow = fl.snk_f[i];
      else for (int v = 0; v < n; ++v) outflow += fl.fc(I, s, i, v);
      if (inflow != g || outflow != g) return 4;  // conservation
    }
  if (fsrc != F || fsnk != F || F > I.M) return 5;
  if (c != cost) return 6;
  Graph G(I, fl);
  const int N = G.N();
  std::vector<Arc> arcs;
  if (F < I.M) {  // maximum: no residual s*-t* path (the reachable set is a cut of capacity F)
    std::vector<char> seen(N, 0);
    std::vector<int> st{G.sstar()};
    seen[G.sstar()] = 1;
    while (!st.empty()) {
      int u = st.back(); st.pop_back();
      G.out_arcs(u, arcs);
      for (const Arc& a : arcs) if (!seen[a.other]) { seen[a.other] = 1; st.push_back(a.other); }
    }
    if (seen[G.tstar()]) return 7;
  }
  // optimal: Bellman-Ford from a virtual root (0 to every node); convergence = no negative cycle
  std::vector<int64_t> pi(N, 0);
  bool changed = true;
  for (int it = 0; it <= N && changed; ++it) {
    changed = false;
    for (int u = 0; u < N; ++u) {
      G.out_arcs(u, arcs);
      for (const Arc& a : arcs)
        if (pi[u] + a.cost < pi[a.other]) { pi[a.other] = pi[u] + a.cost; changed = true; }
    }
  }
  if (changed) return 8;
  for (int u = 0; u < N; ++u) {  // complementary slackness: reduced costs >= 0 on residual arcs
    G.out_arcs(u, arcs);
    for (const Arc& a : arcs) if (a.cost + pi[u] - pi[a.other] < 0) return 9;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Annealing thresholds ("probability e^{(cost_current-cost_new)/T} > U(0,1)",
// "T reduced after each accepted change by a factor alpha")
// ---------------------------------------------------------------------------
uint32_t thr_value(double T0, double alpha, int k, int delta) {
  const double T = T0 * std::pow(alpha, (double)k);
  const double v = std::floor(std::exp(-(double)delta / T) * 4294967296.0);
  if (v >= 4294967295.0) return 4294967295u;
  if (v <= 0.0) return 0u;
  return (uint32_t)v;
}

struct Anneal {
  int32_t width = 1, K = 0;
  std::vector<uint32_t> t;  // (K+1) x width
  int init(double T0, double alpha) {
    if (!(T0 > 0.0)) { width = 1; K = 0; t.assign(1, 0); return 0; }
    if (!(alpha > 0.0 && alpha < 1.0)) return -1;
    width = 1;
    while (thr_value(T0, alpha, 0, width) != 0) { if (++width > (1 << 20)) return -2; }
    K = 0;
    while (thr_value(T0, alpha, K, 1) != 0) { if (++K > (1 << 16)) return -3; }
    if ((int64_t)(K + 1) * width > (1 << 24)) return -4;
    t.assign((size_t)(K + 1) * width, 0);
    for (int k = 0; k <= K; ++k)
      for (int d = 1; d < width; ++d) t[(size_t)k * width + d] = thr_value(T0, alpha, k, d);
    return 0;
  }
  uint32_t get(int k, int64_t delta) const {
    if (delta <= 0 || delta >= width) return 0;
    return t[(size_t)std::min(k, K) * width + delta];
  }
};

// ---------------------------------------------------------------------------
// Decentralized rounds, GWTF-SYNC
// ---------------------------------------------------------------------------
enum { FREE = 0, OUT = 1, IN = 2, PAIRED = 3 };
constexpr int32_t NONE = -1;  // pointers: >=0 relay slot gid*MC+j; NONE; <= -2 data-node slot k = -2-p

uint64_t mix64(uint64_t z) {  // splitmix64 finalizer
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint32_t pick(uint64_t x, uint32_t m) { return (uint32_t)(((x >> 32) * (uint64_t)m) >> 32); }

struct Proposal {
  int kind = 0;  // 0 none, 1 CHANGE, 2 REDIRECT, 3 DENY
  int gid = -1;
  uint64_t key = 0;
  std::vector<int64_t> touched;  // reservation ids
  int32_t x = NONE, y = NONE, z = NONE;
};

struct Rounds {
  Inst I;
  uint64_t seed = 0;
  int64_t inst = 0;
  int obj = 0, W = 5, deny_after = 3;
  Anneal ann;
  std::vector<int32_t> up, down, src_down, snk_up, kacc, deny;
  int32_t quiet = 0;
  int64_t round = 0;

  int Sn() const { return I.S * I.n; }
  int stage(int gid) const { return gid / I.n; }
  int capE(int gid) const { return I.capE(gid / I.n, gid % I.n); }
  bool alive(int gid) const { return I.alive[gid] != 0; }
  int slot(int gid, int j) const { return gid * I.MC + j; }
  static int state_of(int32_t u, int32_t d) {
    return (u != NONE ? 2 : 0) | (d != NONE ? 1 : 0);  // FREE 0, OUT 1, IN 2, PAIRED 3
  }
  int st(int p) const { return state_of(up[p], down[p]); }

  void reset_state() {
    const size_t ns = (size_t)Sn() * I.MC;
    up.assign(ns, NONE);
    down.assign(ns, NONE);
    src_down.assign((size_t)I.M, NONE);
    snk_up.assign((size_t)I.M, NONE);
    kacc.assign(Sn(), 0);
    deny.assign(Sn(), 0);
    quiet = 0;
    round = 0;
  }

  // d(a, b) between nodes; node -1 = data node D.  ABSENT / impossible = INF.
  int64_t d(int a, int b) const {
    int32_t c = ABSENT;
    if (a == -1 && b >= 0 && stage(b) == 0) c = I.src[b % I.n];
    else if (b == -1 && a >= 0 && stage(a) == I.S - 1) c = I.snk[a % I.n];
    else if (a >= 0 && b >= 0 && stage(b) == stage(a) + 1) c = I.C(stage(a), b % I.n, a % I.n);
    return c == ABSENT ? INF : (int64_t)c;
  }
  static int64_t sadd(int64_t a, int64_t b) { return (a == INF || b == INF) ? INF : a + b; }
  int node_of_up(int32_t p) const { return p >= 0 ? p / I.MC : -1; }    // upstream: relay or D (SRC)
  int node_of_down(int32_t p) const { return p >= 0 ? p / I.MC : -1; }  // downstream: relay or D (SNK)

  // R0: cost to sink of every usable slot, back to front
  std::vector<int64_t> costs() const {
    std::vector<int64_t> c((size_t)Sn() * I.MC, INF);
    for (int s = I.S - 1; s >= 0; --s)
      for (int i = 0; i < I.n; ++i) {
        const int v = s * I.n + i;
        for (int j = 0; j < capE(v); ++j) {
          const int p = slot(v, j);
          if (down[p] == NONE) c[p] = INF;
          else if (down[p] <= -2) c[p] = d(v, -1);
          else c[p] = sadd(d(v, down[p] / I.MC), c[down[p]]);
        }
      }
    return c;
  }
  // adv(v) = (min cost over v's OUT slots, lowest slot); INF if none
  std::pair<int64_t, int> adv(int v, const std::vector<int64_t>& c) const {
    std::pair<int64_t, int> best{INF, -1};
    if (!alive(v)) return best;
    for (int j = 0; j < capE(v); ++j) {
      const int p = slot(v, j);
      if (st(p) == OUT && (best.second < 0 || c[p] < best.first)) best = {c[p], j};
    }
    return best;
  }
  uint64_t h(int gid, int stream) const {
    return mix64(mix64(mix64(mix64(seed) ^ (uint64_t)inst) ^ (uint64_t)round) ^ ((uint64_t)gid * 4 + stream));
  }
  int64_t res_id_up(int32_t p) const { return p >= 0 ? p : (int64_t)Sn() * I.MC + (-2 - p); }            // SRC k
  int64_t res_id_down(int32_t p) const { return p >= 0 ? p : (int64_t)Sn() * I.MC + I.M + (-2 - p); }   // SNK k
  void set_up_of(int32_t p, int32_t val) { if (p >= 0) up[p] = val; else snk_up[-2 - p] = val; }      // p is a down pointer
  void set_down_of(int32_t p, int32_t val) { if (p >= 0) down[p] = val; else src_down[-2 - p] = val; }  // p is an up pointer

  uint64_t digest() const {
    uint64_t dg = 0, pos = 0;
    auto add = [&](uint64_t val) { dg += mix64(mix64(pos) ^ val); ++pos; };
    auto enc_up = [&](int32_t p) -> uint64_t { return p == NONE ? 0 : p >= 0 ? 1 + (uint64_t)p : (1ull << 40) + (uint64_t)(-2 - p); };
    auto enc_dn = [&](int32_t p) -> uint64_t { return p == NONE ? 0 : p >= 0 ? 1 + (uint64_t)p : (1ull << 41) + (uint64_t)(-2 - p); };
    for (size_t p = 0; p < up.size(); ++p) { add((uint64_t)st((int)p)); add(enc_up(up[p])); add(enc_dn(down[p])); }
    for (int64_t k = 0; k < I.M; ++k) add(src_down[k] == NONE ? 0 : 1 + (uint64_t)src_down[k]);
    for (int64_t k = 0; k < I.M; ++k) add(snk_up[k] == NONE ? 0 : 1 + (uint64_t)snk_up[k]);
    for (int g = 0; g < Sn(); ++g) { add((uint64_t)(uint32_t)kacc[g]); add((uint64_t)(uint32_t)deny[g]); }
    add((uint64_t)(uint32_t)quiet);
    return dg;
  }

  // one synchronous round; returns the number of structural changes
  int64_t one_round() {
    const int S = I.S, n = I.n, Sn_ = Sn();
    int64_t changes = 0;
    // R0a self-pairing, costs from the round-start state
    {
      const std::vector<int64_t> c0 = costs();
      for (int v = 0; v < Sn_; ++v) {
        if (!alive(v)) continue;
        int x = -1, o = -1;
        for (int j = 0; j < capE(v); ++j) {
          const int p = slot(v, j);
          if (x < 0 && st(p) == IN) x = p;
          if (st(p) == OUT && (o < 0 || c0[p] < c0[o])) o = p;
        }
        if (x < 0 || o < 0) continue;
        const int32_t cdn = down[o];
        down[x] = cdn;
        set_up_of(cdn, x);
        down[o] = NONE;
        ++changes;
      }
    }
    // R0 costs and advertisements on the post-R0a state
    const std::vector<int64_t> c = costs();
    std::vector<std::pair<int64_t, int>> ad(Sn_);
    for (int v = 0; v < Sn_; ++v) ad[v] = adv(v, c);
    bool dsink_free = false;
    for (int64_t k = 0; k < I.M; ++k) if (snk_up[k] == NONE) { dsink_free = true; break; }
    // R1 requests: requester slot and target node (-1 = D-sink) of every relay, and of D
    std::vector<int32_t> rslot(Sn_, NONE), target(Sn_, -2);
    std::vector<char> requested(Sn_, 0);
    for (int r = 0; r < Sn_; ++r) {
      if (!alive(r)) continue;
      int xin = -1, xfree = -1;
      bool has_out = false;
      for (int j = 0; j < capE(r); ++j) {
        const int p = slot(r, j), t = st(p);
        if (t == IN && xin < 0) xin = p;
        if (t == FREE && xfree < 0) xfree = p;
        if (t == OUT) has_out = true;
      }
      int32_t rs = NONE;
      if (xin >= 0) rs = xin;                       // (a) unpaired inflow
      else if (!has_out && xfree >= 0) rs = xfree;  // (b) stable with spare capacity
      if (rs == NONE) continue;
      const int s = stage(r);
      int best = -2;
      int64_t bestc = INF;
      if (s == S - 1) {
        if (d(r, -1) != INF && dsink_free) { best = -1; bestc = d(r, -1); }
      } else {
        for (int jj = 0; jj < n; ++jj) {
          const int j = (s + 1) * n + jj;
          if (!alive(j) || d(r, j) == INF || ad[j].first == INF) continue;
          const int64_t tc = d(r, j) + ad[j].first;
          if (tc < bestc) { bestc = tc; best = j; }
        }
      }
      if (best == -2) continue;  // no target: idle
      rslot[r] = rs;
      target[r] = best;
      requested[r] = 1;
    }
    int64_t d_rslot = -1;
    int d_target = -2;
    for (int64_t k = 0; k < I.M; ++k) if (src_down[k] == NONE) { d_rslot = k; break; }
    if (d_rslot >= 0) {
      int64_t bestc = INF;
      for (int j = 0; j < n; ++j)
        if (alive(j) && d(-1, j) != INF && ad[j].first != INF && d(-1, j) + ad[j].first < bestc) {
          bestc = d(-1, j) + ad[j].first;
          d_target = j;
        }
    }
    // R2 grants (requesters in ascending gid, D first) + R3 commit
    {
      // relay targets
      std::vector<int> rank_count(Sn_, 0);
      auto eligible = [&](int j, int q) -> int32_t {  // q-th OUT slot of j with cost == adv(j)
        int cnt = 0;
        for (int jj = 0; jj < capE(j); ++jj) {
          const int p = slot(j, jj);
          if (st(p) == OUT && c[p] == ad[j].first) { if (cnt == q) return p; ++cnt; }
        }
        return NONE;
      };
      struct Grant { int req; int32_t rs; int32_t ts; };
      std::vector<Grant> grants;
      if (d_target >= 0) {  // D orders before all relays
        const int32_t ts = eligible(d_target, rank_count[d_target]++);
        if (ts != NONE) grants.push_back({-1, (int32_t)(-2 - d_rslot), ts});
      }
      std::vector<int> snk_free;
      for (int64_t k = 0; k < I.M; ++k) if (snk_up[k] == NONE) snk_free.push_back((int)k);
      size_t snk_rank = 0;
      for (int r = 0; r < Sn_; ++r) {
        if (!requested[r]) continue;
        if (target[r] == -1) {
          if (snk_rank < snk_free.size()) grants.push_back({r, rslot[r], (int32_t)(-2 - snk_free[snk_rank])});
          ++snk_rank;
        } else {
          const int32_t ts = eligible(target[r], rank_count[target[r]]++);
          if (ts != NONE) grants.push_back({r, rslot[r], ts});
        }
      }
      for (const Grant& gr : grants) {
        if (gr.req == -1) src_down[-2 - gr.rs] = gr.ts;  // SRC k -> relay slot
        else { down[gr.rs] = gr.ts; deny[gr.req] = 0; }
        // the granted slot (relay OUT slot or SNK k) gets its upstream
        if (gr.ts >= 0) up[gr.ts] = gr.rs;
        else snk_up[-2 - gr.ts] = gr.rs;
        ++changes;
      }
    }
    // R4 move proposals by idle relays (post-R3 state)
    std::vector<Proposal> props;
    for (int p = 0; p < Sn_; ++p) {
      if (!alive(p) || requested[p]) continue;
      const int s = stage(p), i = p % n;
      int xin = -1, zfree = -1;
      bool has_out = false;
      std::vector<int> P;
      for (int j = 0; j < capE(p); ++j) {
        const int q = slot(p, j), t = st(q);
        if (t == IN && xin < 0) xin = q;
        if (t == FREE && zfree < 0) zfree = q;
        if (t == OUT) has_out = true;
        if (t == PAIRED) P.push_back(q);
      }
      if (xin >= 0) {  // DENY after deny_after idle rounds holding unpaired inflow
        deny[p] += 1;
        if (deny[p] >= deny_after) {
          Proposal pr;
          pr.kind = 3; pr.gid = p; pr.key = ((uint64_t)0 << 22) | (uint64_t)p;  // delta = -inf
          pr.x = xin;
          pr.touched = {xin, res_id_up(up[xin])};
          props.push_back(pr);
        }
        continue;
      }
      if (n < 2) continue;
      uint32_t qi = pick(h(p, 0), (uint32_t)(n - 1));
      if ((int)qi >= i) qi += 1;
      const int q = s * n + (int)qi;
      if (!alive(q)) continue;
      std::vector<int> Q;
      for (int j = 0; j < capE(q); ++j) if (st(slot(q, j)) == PAIRED) Q.push_back(slot(q, j));
      if (Q.empty()) continue;
      Proposal pr;
      pr.gid = p;
      int64_t delta;
      if (zfree >= 0 && !has_out) {  // Request Redirect
        const int y = Q[pick(h(p, 2), (uint32_t)Q.size())];
        const int a = node_of_up(up[y]), cc = node_of_down(down[y]), b = q;
        const int64_t dax = d(a, p), dxc = d(p, cc), dab = d(a, b), dbc = d(b, cc);
        if (dax == INF || dxc == INF || dab == INF || dbc == INF) continue;
        delta = (obj == ORC_OBJ_SUM) ? (dax + dxc) - (dab + dbc) : std::max(dax, dxc) - std::max(dab, dbc);
        pr.kind = 2; pr.y = y; pr.z = zfree;
        pr.touched = {y, res_id_up(up[y]), res_id_down(down[y]), zfree};
      } else if (!P.empty()) {  // Request Change
        const int x = P[pick(h(p, 1), (uint32_t)P.size())];
        const int y = Q[pick(h(p, 2), (uint32_t)Q.size())];
        const int j1 = node_of_down(down[x]), j2 = node_of_down(down[y]);
        if (j1 == j2) continue;
        const int64_t dpj2 = d(p, j2), dqj1 = d(q, j1), dpj1 = d(p, j1), dqj2 = d(q, j2);
        if (dpj2 == INF || dqj1 == INF || dpj1 == INF || dqj2 == INF) continue;
        delta = (obj == ORC_OBJ_SUM) ? (dpj2 + dqj1) - (dpj1 + dqj2) : std::max(dpj2, dqj1) - std::max(dpj1, dqj2);
        pr.kind = 1; pr.x = x; pr.y = y;
        pr.touched = {x, y, res_id_down(down[x]), res_id_down(down[y])};
      } else {
        continue;
      }
      if (delta == 0) continue;  // equal-cost moves are never proposed
      if (delta > 0 && !((h(p, 3) >> 32) < (uint64_t)ann.get(kacc[p], delta))) continue;
      pr.key = ((uint64_t)(delta + (1ll << 40)) << 22) | (uint64_t)p;
      props.push_back(pr);
    }
    // R5 deterministic reservations: min key per touched slot
    const int64_t nres = (int64_t)Sn_ * I.MC + 2 * I.M;
    std::vector<uint64_t> res((size_t)nres, UINT64_MAX);
    for (const Proposal& pr : props)
      for (int64_t t : pr.touched) res[t] = std::min(res[t], pr.key);
    // R6 commit the proposals that hold every slot they touch
    for (const Proposal& pr : props) {
      bool win = true;
      for (int64_t t : pr.touched) win = win && res[t] == pr.key;
      if (!win) continue;
      if (pr.kind == 1) {  // Change: swap the down pointers of x and y
        const int32_t dx = down[pr.x], dy = down[pr.y];
        down[pr.x] = dy; down[pr.y] = dx;
        set_up_of(dy, pr.x);
        set_up_of(dx, pr.y);
        kacc[pr.gid] += 1;
      } else if (pr.kind == 2) {  // Redirect: z takes (up, down) of y; y becomes FREE
        const int32_t a = up[pr.y], cc = down[pr.y];
        up[pr.z] = a; down[pr.z] = cc;
        set_down_of(a, pr.z);
        set_up_of(cc, pr.z);
        up[pr.y] = NONE; down[pr.y] = NONE;
        kacc[pr.gid] += 1;
      } else if (pr.kind == 3) {  // DENY: own IN slot freed, upstream loses its downstream
        const int32_t a = up[pr.x];
        up[pr.x] = NONE;
        set_down_of(a, NONE);
        deny[pr.gid] = 0;
      }
      ++changes;
    }
    // R7 bookkeeping
    quiet = changes > 0 ? 0 : quiet + 1;
    round += 1;
    return changes;
  }

  void result(int64_t* F_dec, int64_t* cost_dec, int32_t* dangling) const {
    int64_t F = 0, C = 0;
    for (int64_t k = 0; k < I.M; ++k) {
      int32_t p = src_down[k];
      if (p == NONE) continue;
      int64_t cc = d(-1, p / I.MC);
      int guard = 0;
      while (p >= 0 && ++guard <= I.S + 1) {
        const int32_t nx = down[p];
        if (nx == NONE) { cc = -1; break; }
        cc = sadd(cc, nx <= -2 ? d(p / I.MC, -1) : d(p / I.MC, nx / I.MC));
        p = nx;
      }
      if (cc >= 0 && cc != INF && p <= -2) { F += 1; C += cc; }
    }
    int32_t dang = 0;
    for (size_t p = 0; p < up.size(); ++p) if (st((int)p) == OUT) ++dang;
    *F_dec = F; *cost_dec = C; *dangling = dang;
  }

  // order-independent pointer clearing
  void apply_churn(const uint8_t* alive_new, const int32_t* upd, int64_t k) {
    const int S = I.S, n = I.n;
    for (int64_t e = 0; e < k; ++e) {
      const int32_t* u = upd + 5 * e;
      const int s = u[1], v = u[2], w = u[3];
      if (s == -1) I.src[v] = u[4];
      else if (s == S - 1) I.snk[w] = u[4];
      else I.Cref(s, v, w) = u[4];
    }
    if (alive_new) for (int g = 0; g < S * n; ++g) I.alive[g] = alive_new[g];
    auto dead_or_beyond = [&](int32_t p) { return p >= 0 && (!alive(p / I.MC) || p % I.MC >= capE(p / I.MC)); };
    for (int v = 0; v < S * n; ++v)
      for (int j = 0; j < I.MC; ++j) {
        const int p = slot(v, j);
        if (!alive(v) || j >= capE(v)) { up[p] = NONE; down[p] = NONE; continue; }
        if (up[p] != NONE) {
          const int a = node_of_up(up[p]);
          if ((up[p] >= 0 && dead_or_beyond(up[p])) || d(a, v) == INF) up[p] = NONE;
        }
        if (down[p] != NONE) {
          const int c = node_of_down(down[p]);
          if ((down[p] >= 0 && dead_or_beyond(down[p])) || d(v, c) == INF) down[p] = NONE;
        }
      }
    for (int64_t kk = 0; kk < I.M; ++kk) {
      const int32_t p = src_down[kk];
      if (p != NONE && (dead_or_beyond(p) || d(-1, p / I.MC) == INF)) src_down[kk] = NONE;
      const int32_t q = snk_up[kk];
      if (q != NONE && (dead_or_beyond(q) || d(q / I.MC, -1) == INF)) snk_up[kk] = NONE;
    }
    std::fill(kacc.begin(), kacc.end(), 0);
    std::fill(deny.begin(), deny.end(), 0);
    quiet = 0;
  }
};

template <class Fn>
void parallel_for(int64_t B, int threads, Fn fn) {
  if (threads <= 1 || B <= 1) {
    for (int64_t b = 0; b < B; ++b) fn(b);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&]() {
      for (int64_t b; (b = next.fetch_add(1)) < B;) fn(b);
    });
  for (auto& th : pool) th.join();
}

orc_instance view(int64_t b, int32_t S, int32_t n, int32_t max_cap, const int32_t* cap, const uint8_t* alive,
                  const int32_t* src, const int32_t* snk, const int32_t* link, const int64_t* supply) {
  orc_instance I;
  I.S = S; I.n = n; I.max_cap = max_cap; I.M = supply[b];
  I.cap = cap + b * S * n;
  I.alive = alive ? alive + b * S * n : nullptr;
  I.src = src + b * n;
  I.snk = snk + b * n;
  I.link = link + b * (int64_t)std::max(S - 1, 0) * n * n;
  return I;
}

// ---------------------------------------------------------------------------
// Warm-start rerouting after churn ("reroute",
// :274-288 crash handling).  Textbook steps, in order:
//   1. keep the pre-churn flow; strip every unit that crosses a crashed relay,
//      a relay over its new capacity, or a link/src/snk whose new cost is ABSENT
//      (one unit path at a time, lowest-index predecessor / successor first);
//   2. cancel negative residual cycles (Klein): Bellman-Ford from a virtual root,
//      a relaxation in pass N proves a cycle, walk the predecessors into it and
//      push its bottleneck; repeat until none;
//   3. resume successive shortest paths (Bellman-Ford on the residual graph,
//      which has no negative cycle after 2) until F = M or t* is unreachable.
// Explicit arc list; shares nothing with ssp() above, so it can pin it.
// ---------------------------------------------------------------------------
struct WArc { int from, to; int64_t cap, cost, x; };

struct WarmGraph {
  int S, n, N;
  std::vector<WArc> A;
  int sstar() const { return 0; }
  int tstar() const { return 1; }
  int in(int s, int i) const { return 2 + 2 * (s * n + i); }
  int out(int s, int i) const { return 3 + 2 * (s * n + i); }
  std::vector<int> src_arc, snk_arc, node_arc, link_arc;  // -1 = absent
  explicit WarmGraph(const Inst& I) : S(I.S), n(I.n), N(2 + 2 * I.S * I.n) {
    const int64_t U = I.M;  // no path carries more than the supply
    src_arc.assign(n, -1); snk_arc.assign(n, -1); node_arc.assign((size_t)S * n, -1);
    link_arc.assign(S > 1 ? (size_t)(S - 1) * n * n : 0, -1);
    for (int i = 0; i < n; ++i)
      if (I.src[i] != ABSENT) { src_arc[i] = (int)A.size(); A.push_back({sstar(), in(0, i), U, I.src[i], 0}); }
    for (int s = 0; s < S; ++s)
      for (int i = 0; i < n; ++i) {
        node_arc[(size_t)s * n + i] = (int)A.size();
        A.push_back({in(s, i), out(s, i), I.capE(s, i), 0, 0});
      }
    for (int s = 0; s + 1 < S; ++s)
      for (int v = 0; v < n; ++v)
        for (int u = 0; u < n; ++u)
          if (I.C(s, v, u) != ABSENT) {
            link_arc[((size_t)s * n + v) * n + u] = (int)A.size();
            A.push_back({out(s, u), in(s + 1, v), U, I.C(s, v, u), 0});
          }
    for (int i = 0; i < n; ++i)
      if (I.snk[i] != ABSENT) { snk_arc[i] = (int)A.size(); A.push_back({out(S - 1, i), tstar(), U, I.snk[i], 0}); }
  }
  // residual arc r: r = 2e forward (cap - x, +cost), r = 2e+1 backward (x, -cost)
  int64_t rcap(int r) const { const WArc& a = A[r >> 1]; return (r & 1) ? a.x : a.cap - a.x; }
  int64_t rcost(int r) const { return (r & 1) ? -A[r >> 1].cost : A[r >> 1].cost; }
  int rfrom(int r) const { return (r & 1) ? A[r >> 1].to : A[r >> 1].from; }
  int rto(int r) const { return (r & 1) ? A[r >> 1].from : A[r >> 1].to; }
  void push(int r, int64_t d) { if (r & 1) A[r >> 1].x -= d; else A[r >> 1].x += d; }
};

// Step 1 helper: remove one unit along a path through arc e (upstream then downstream).
// Every arc strictly inside the layered graph has an upstream/downstream path with flow
// because the pre-churn flow is conserved.
void warm_strip_unit(WarmGraph& G, int e) {
  std::vector<int> path{e};
  for (int node = G.A[e].from; node != G.sstar();) {  // upstream: lowest-index arc into node with flow
    int pick = -1;
    for (int k = 0; k < (int)G.A.size() && pick < 0; ++k)
      if (G.A[k].to == node && G.A[k].x > 0) pick = k;
    path.push_back(pick);
    node = G.A[pick].from;
  }
  for (int node = G.A[e].to; node != G.tstar();) {  // downstream: lowest-index arc out of node with flow
    int pick = -1;
    for (int k = 0; k < (int)G.A.size() && pick < 0; ++k)
      if (G.A[k].from == node && G.A[k].x > 0) pick = k;
    path.push_back(pick);
    node = G.A[pick].to;
  }
  for (int k : path) G.A[k].x -= 1;
}

struct WarmStats { int64_t stripped = 0, cycles = 0, augment = 0; };

int warm_reroute(const Inst& Iold, const Flow& fold, const Inst& Inew, Flow& out, WarmStats& st) {
  const int S = Inew.S, n = Inew.n;
  WarmGraph G(Inew);
  // Step 1: carry the old flow over.  Arcs that vanished (ABSENT) or relays with less
  // capacity keep their old flow first on a temporary arc so that it can be stripped.
  const size_t nbase = G.A.size();
  auto carry = [&](int e_new, int64_t x, int from, int to, int64_t cost_old) -> int {
    if (x == 0) return 0;
    if (e_new < 0) {  // vanished arc: a temporary zero-capacity copy holding the old flow
      G.A.push_back({from, to, 0, cost_old, x});
      return 0;
    }
    G.A[e_new].x = x;
    return 0;
  };
  for (int i = 0; i < n; ++i) {
    carry(G.src_arc[i], fold.src_f[i], G.sstar(), G.in(0, i), Iold.src[i]);
    carry(G.snk_arc[i], fold.snk_f[i], G.out(S - 1, i), G.tstar(), Iold.snk[i]);
  }
  for (int s = 0; s < S; ++s)
    for (int i = 0; i < n; ++i) carry(G.node_arc[(size_t)s * n + i], fold.g[(size_t)s * n + i], G.in(s, i), G.out(s, i), 0);
  for (int s = 0; s + 1 < S; ++s)
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u)
        carry(G.link_arc[((size_t)s * n + v) * n + u], fold.fc(Iold, s, u, v), G.out(s, u), G.in(s + 1, v), Iold.C(s, v, u));
  for (int e = 0; e < (int)G.A.size(); ++e)
    while (G.A[e].x > G.A[e].cap) { warm_strip_unit(G, e); ++st.stripped; }
  for (size_t e = nbase; e < G.A.size(); ++e)
    if (G.A[e].x != 0) return -31;
  G.A.resize(nbase);  // the temporary arcs are empty now
  const int N = G.N, R = 2 * (int)G.A.size();
  // Step 2: negative-cycle cancelling
  for (;;) {
    std::vector<int64_t> d(N, 0);
    std::vector<int> pred(N, -1);
    int last = -1;
    for (int pass = 0; pass < N; ++pass) {
      last = -1;
      for (int r = 0; r < R; ++r)
        if (G.rcap(r) > 0 && d[G.rfrom(r)] + G.rcost(r) < d[G.rto(r)]) {
          d[G.rto(r)] = d[G.rfrom(r)] + G.rcost(r);
          pred[G.rto(r)] = r;
          last = G.rto(r);
        }
      if (last < 0) break;
    }
    if (last < 0) break;
    int x = last;
    for (int k = 0; k < N; ++k) x = G.rfrom(pred[x]);  // now on the cycle
    std::vector<int> cyc;
    int y = x;
    do { cyc.push_back(pred[y]); y = G.rfrom(pred[y]); } while (y != x);
    int64_t b = INF;
    for (int r : cyc) b = std::min(b, G.rcap(r));
    for (int r : cyc) G.push(r, b);
    ++st.cycles;
  }
  // Step 3: successive shortest paths from the cancelled flow
  int64_t F = 0;
  for (int i = 0; i < n; ++i) if (G.src_arc[i] >= 0) F += G.A[G.src_arc[i]].x;
  while (F < Inew.M) {
    std::vector<int64_t> d(N, INF);
    std::vector<int> pred(N, -1);
    d[G.sstar()] = 0;
    for (int pass = 0; pass < N; ++pass) {
      bool ch = false;
      for (int r = 0; r < R; ++r)
        if (G.rcap(r) > 0 && d[G.rfrom(r)] != INF && d[G.rfrom(r)] + G.rcost(r) < d[G.rto(r)]) {
          d[G.rto(r)] = d[G.rfrom(r)] + G.rcost(r);
          pred[G.rto(r)] = r;
          ch = true;
        }
      if (!ch) break;
    }
    if (d[G.tstar()] == INF) break;
    int64_t b = Inew.M - F;
    for (int v = G.tstar(); v != G.sstar(); v = G.rfrom(pred[v])) b = std::min(b, G.rcap(pred[v]));
    for (int v = G.tstar(); v != G.sstar(); v = G.rfrom(pred[v])) G.push(pred[v], b);
    F += b;
    ++st.augment;
  }
  // assignment out
  out.F = F; out.cost = 0; out.A = (int32_t)st.augment;
  for (const WArc& a : G.A) out.cost += a.x * a.cost;
  for (int i = 0; i < n; ++i) {
    out.src_f[i] = G.src_arc[i] >= 0 ? (int32_t)G.A[G.src_arc[i]].x : 0;
    out.snk_f[i] = G.snk_arc[i] >= 0 ? (int32_t)G.A[G.snk_arc[i]].x : 0;
  }
  for (int k = 0; k < S * n; ++k) out.g[k] = (int32_t)G.A[G.node_arc[k]].x;
  for (size_t k = 0; k < G.link_arc.size(); ++k) out.arc[k] = G.link_arc[k] >= 0 ? (int32_t)G.A[G.link_arc[k]].x : 0;
  return 0;
}

}  // namespace

struct orc_rounds { Rounds R; };
// ---------------------------------------------------------------------------
// Multi-data-node decentralized rounds, MC-SYNC.
// "each data node ... must receive its own flow back", :209, settings 5-6 of :501-502.  K data
// nodes D_0..D_{K-1}, each with its own supply M_k, SRC_k / SNK_k slots and source / sink costs;
// the relays and links are shared.  Every non-FREE relay slot carries the data node (tag) of its
// chain: an OUT slot of tag k is "unpaired outflow to data node k", so requests, grants,
// swaps and self-pairing stay within one tag.  With K = 1 every rule is the single-commodity one.
// Pointers: relay slot >= 0, NONE, data-node slot -2 - (k * Mmax + i).
// ---------------------------------------------------------------------------
struct McRounds {
  Inst I;
  int K = 1;
  int64_t Mmax = 0;
  std::vector<int64_t> M;                  // [K]
  std::vector<int32_t> srcK, snkK;         // [K][n]
  uint64_t seed = 0;
  int64_t inst = 0;
  int obj = 0, W = 5, deny_after = 3;
  Anneal ann;
  std::vector<int32_t> up, down, tag, src_down, snk_up, kacc, deny;  // src_down / snk_up [K][Mmax]
  int32_t quiet = 0;
  int64_t round = 0;

  int Sn() const { return I.S * I.n; }
  int stage(int gid) const { return gid / I.n; }
  int capE(int gid) const { return I.capE(gid / I.n, gid % I.n); }
  bool alive(int gid) const { return I.alive[gid] != 0; }
  int slot(int gid, int j) const { return gid * I.MC + j; }
  int st(int p) const { return Rounds::state_of(up[p], down[p]); }
  static int32_t dptr(int k, int64_t i, int64_t Mm) { return (int32_t)(-2 - (k * Mm + i)); }
  int dk(int32_t p) const { return (int)((-2 - (int64_t)p) / Mmax); }   // data node of a data-node pointer
  int64_t di(int32_t p) const { return (-2 - (int64_t)p) % Mmax; }      // its slot index

  void reset_state() {
    const size_t ns = (size_t)Sn() * I.MC;
    up.assign(ns, NONE); down.assign(ns, NONE); tag.assign(ns, 0);
    src_down.assign((size_t)K * Mmax, NONE); snk_up.assign((size_t)K * Mmax, NONE);
    kacc.assign(Sn(), 0); deny.assign(Sn(), 0);
    quiet = 0; round = 0;
  }
  // d(a, b); node -1-k = data node k (SRC side for a, SNK side for b)
  int64_t d(int a, int b) const {
    int32_t c = ABSENT;
    if (a < 0 && b >= 0 && stage(b) == 0) c = srcK[(size_t)(-1 - a) * I.n + b % I.n];
    else if (b < 0 && a >= 0 && stage(a) == I.S - 1) c = snkK[(size_t)(-1 - b) * I.n + a % I.n];
    else if (a >= 0 && b >= 0 && stage(b) == stage(a) + 1) c = I.C(stage(a), b % I.n, a % I.n);
    return c == ABSENT ? INF : (int64_t)c;
  }
  int node_of(int32_t p) const { return p >= 0 ? p / I.MC : -1 - dk(p); }  // relay or data node (-1-k)
  void set_up_of(int32_t p, int32_t v) { if (p >= 0) up[p] = v; else snk_up[(size_t)dk(p) * Mmax + di(p)] = v; }
  void set_down_of(int32_t p, int32_t v) { if (p >= 0) down[p] = v; else src_down[(size_t)dk(p) * Mmax + di(p)] = v; }
  int64_t res_id_up(int32_t p) const { return p >= 0 ? p : (int64_t)Sn() * I.MC + (-2 - (int64_t)p); }
  int64_t res_id_down(int32_t p) const { return p >= 0 ? p : (int64_t)Sn() * I.MC + (int64_t)K * Mmax + (-2 - (int64_t)p); }
  uint64_t h(int gid, int stream) const {
    return mix64(mix64(mix64(mix64(seed) ^ (uint64_t)inst) ^ (uint64_t)round) ^ ((uint64_t)gid * 4 + stream));
  }

  std::vector<int64_t> costs() const {  // R0, back to front
    std::vector<int64_t> c((size_t)Sn() * I.MC, INF);
    for (int s = I.S - 1; s >= 0; --s)
      for (int i = 0; i < I.n; ++i) {
        const int v = s * I.n + i;
        for (int j = 0; j < capE(v); ++j) {
          const int p = slot(v, j);
          if (down[p] == NONE) c[p] = INF;
          else if (down[p] <= -2) c[p] = d(v, -1 - dk(down[p]));
          else c[p] = Rounds::sadd(d(v, down[p] / I.MC), c[down[p]]);
        }
      }
    return c;
  }
  // adv(v, k) = min cost over v's OUT slots of tag k (INF if none)
  int64_t adv(int v, int k, const std::vector<int64_t>& c) const {
    int64_t best = INF;
    if (!alive(v)) return best;
    for (int j = 0; j < capE(v); ++j) {
      const int p = slot(v, j);
      if (st(p) == OUT && tag[p] == k && c[p] < best) best = c[p];
    }
    return best;
  }
  bool sink_free(int k) const {
    for (int64_t i = 0; i < M[k]; ++i) if (snk_up[(size_t)k * Mmax + i] == NONE) return true;
    return false;
  }

  int64_t one_round() {
    const int S = I.S, n = I.n, Sn_ = Sn();
    int64_t changes = 0;
    {  // R0a: the lowest IN slot whose tag has an OUT slot takes its min-(cost, slot) OUT slot's downstream
      const std::vector<int64_t> c0 = costs();
      for (int v = 0; v < Sn_; ++v) {
        if (!alive(v)) continue;
        int x = -1, o = -1;
        for (int j = 0; j < capE(v) && x < 0; ++j) {
          const int p = slot(v, j);
          if (st(p) != IN) continue;
          int ob = -1;
          for (int jj = 0; jj < capE(v); ++jj) {
            const int q = slot(v, jj);
            if (st(q) == OUT && tag[q] == tag[p] && (ob < 0 || c0[q] < c0[ob])) ob = q;
          }
          if (ob >= 0) { x = p; o = ob; }
        }
        if (x < 0) continue;
        const int32_t cdn = down[o];
        down[x] = cdn;
        set_up_of(cdn, x);
        down[o] = NONE;
        ++changes;
      }
    }
    const std::vector<int64_t> c = costs();
    std::vector<int64_t> ad((size_t)Sn_ * K);
    for (int v = 0; v < Sn_; ++v) for (int k = 0; k < K; ++k) ad[(size_t)v * K + k] = adv(v, k, c);
    std::vector<char> sfree(K);
    for (int k = 0; k < K; ++k) sfree[k] = sink_free(k);
    // R1: requests (requester slot, target node or -1-k for D_k-sink, commodity)
    std::vector<int32_t> rslot(Sn_, NONE), target(Sn_, INT32_MIN), rk(Sn_, -1);
    std::vector<char> requested(Sn_, 0);
    for (int r = 0; r < Sn_; ++r) {
      if (!alive(r)) continue;
      int xin = -1, xfree = -1;
      bool has_out = false;
      for (int j = 0; j < capE(r); ++j) {
        const int p = slot(r, j), t = st(p);
        if (t == IN && xin < 0) xin = p;
        if (t == FREE && xfree < 0) xfree = p;
        if (t == OUT) has_out = true;
      }
      int32_t rs = NONE;
      if (xin >= 0) rs = xin;
      else if (!has_out && xfree >= 0) rs = xfree;
      if (rs == NONE) continue;
      const int s = stage(r);
      const int klo = xin >= 0 ? tag[xin] : 0, khi = xin >= 0 ? tag[xin] : K - 1;  // (a) own tag, (b) any
      int best = INT32_MIN, bk = -1;
      int64_t bestc = INF;
      if (s == S - 1) {
        for (int k = klo; k <= khi; ++k)
          if (sfree[k] && d(r, -1 - k) != INF && d(r, -1 - k) < bestc) { bestc = d(r, -1 - k); best = -1 - k; bk = k; }
      } else {
        for (int jj = 0; jj < n; ++jj) {  // lowest j, then lowest k, on ties
          const int j = (s + 1) * n + jj;
          if (!alive(j) || d(r, j) == INF) continue;
          for (int k = klo; k <= khi; ++k) {
            const int64_t a = ad[(size_t)j * K + k];
            if (a == INF) continue;
            if (d(r, j) + a < bestc) { bestc = d(r, j) + a; best = j; bk = k; }
          }
        }
      }
      if (bk < 0) continue;  // no target: idle
      rslot[r] = rs; target[r] = best; rk[r] = bk; requested[r] = 1;
    }
    // data nodes: D_k requests for its lowest unpaired SRC_k slot (stage-0 advertisers of tag k)
    std::vector<int64_t> d_slot(K, -1);
    std::vector<int> d_target(K, -1);
    for (int k = 0; k < K; ++k) {
      for (int64_t i = 0; i < M[k]; ++i) if (src_down[(size_t)k * Mmax + i] == NONE) { d_slot[k] = i; break; }
      if (d_slot[k] < 0) continue;
      int64_t bestc = INF;
      for (int j = 0; j < n; ++j) {
        const int64_t a = ad[(size_t)j * K + k];
        if (alive(j) && d(-1 - k, j) != INF && a != INF && d(-1 - k, j) + a < bestc) { bestc = d(-1 - k, j) + a; d_target[k] = j; }
      }
    }
    // R2 + R3: targets serve D_0..D_{K-1} then relays in gid order, per-tag OUT slots with cost == adv
    {
      std::vector<int> rank((size_t)Sn_ * K, 0);
      auto eligible = [&](int j, int k, int q) -> int32_t {
        int cnt = 0;
        for (int jj = 0; jj < capE(j); ++jj) {
          const int p = slot(j, jj);
          if (st(p) == OUT && tag[p] == k && c[p] == ad[(size_t)j * K + k]) { if (cnt == q) return p; ++cnt; }
        }
        return NONE;
      };
      struct Grant { int req; int k; int32_t rs; int32_t ts; };
      std::vector<Grant> grants;
      for (int k = 0; k < K; ++k)
        if (d_target[k] >= 0) {
          const int j = d_target[k];
          const int32_t ts = eligible(j, k, rank[(size_t)j * K + k]++);
          if (ts != NONE) grants.push_back({-1, k, dptr(k, d_slot[k], Mmax), ts});
        }
      std::vector<size_t> snk_rank(K, 0);
      std::vector<std::vector<int>> snk_free(K);
      for (int k = 0; k < K; ++k)
        for (int64_t i = 0; i < M[k]; ++i) if (snk_up[(size_t)k * Mmax + i] == NONE) snk_free[k].push_back((int)i);
      for (int r = 0; r < Sn_; ++r) {
        if (!requested[r]) continue;
        const int k = rk[r];
        if (target[r] < 0) {
          if (snk_rank[k] < snk_free[k].size()) grants.push_back({r, k, rslot[r], dptr(k, snk_free[k][snk_rank[k]], Mmax)});
          ++snk_rank[k];
        } else {
          const int j = target[r];
          const int32_t ts = eligible(j, k, rank[(size_t)j * K + k]++);
          if (ts != NONE) grants.push_back({r, k, rslot[r], ts});
        }
      }
      for (const Grant& gr : grants) {
        if (gr.req == -1) src_down[(size_t)dk(gr.rs) * Mmax + di(gr.rs)] = gr.ts;
        else { down[gr.rs] = gr.ts; tag[gr.rs] = gr.k; deny[gr.req] = 0; }
        if (gr.ts >= 0) up[gr.ts] = gr.rs;
        else snk_up[(size_t)dk(gr.ts) * Mmax + di(gr.ts)] = gr.rs;
        ++changes;
      }
    }
    // R4 proposals by idle relays (post-R3 state); R5 reservations; R6 commits
    std::vector<Proposal> props;
    for (int p = 0; p < Sn_; ++p) {
      if (!alive(p) || requested[p]) continue;
      const int s = stage(p), i = p % n;
      int xin = -1, zfree = -1;
      bool has_out = false;
      std::vector<int> Pl;
      for (int j = 0; j < capE(p); ++j) {
        const int q = slot(p, j), t = st(q);
        if (t == IN && xin < 0) xin = q;
        if (t == FREE && zfree < 0) zfree = q;
        if (t == OUT) has_out = true;
        if (t == PAIRED) Pl.push_back(q);
      }
      if (xin >= 0) {
        deny[p] += 1;
        if (deny[p] >= deny_after) {
          Proposal pr;
          pr.kind = 3; pr.gid = p; pr.key = (uint64_t)p; pr.x = xin;
          pr.touched = {xin, res_id_up(up[xin])};
          props.push_back(pr);
        }
        continue;
      }
      if (n < 2) continue;
      uint32_t qi = pick(h(p, 0), (uint32_t)(n - 1));
      if ((int)qi >= i) qi += 1;
      const int q = s * n + (int)qi;
      if (!alive(q)) continue;
      std::vector<int> Q;
      for (int j = 0; j < capE(q); ++j) if (st(slot(q, j)) == PAIRED) Q.push_back(slot(q, j));
      if (Q.empty()) continue;
      Proposal pr;
      pr.gid = p;
      int64_t delta;
      if (zfree >= 0 && !has_out) {  // Redirect: z takes y's (up, down, tag)
        const int y = Q[pick(h(p, 2), (uint32_t)Q.size())];
        const int a = node_of(up[y]), cc = node_of(down[y]), b = q;
        const int64_t dax = d(a, p), dxc = d(p, cc), dab = d(a, b), dbc = d(b, cc);
        if (dax == INF || dxc == INF || dab == INF || dbc == INF) continue;
        delta = (obj == ORC_OBJ_SUM) ? (dax + dxc) - (dab + dbc) : std::max(dax, dxc) - std::max(dab, dbc);
        pr.kind = 2; pr.y = y; pr.z = zfree;
        pr.touched = {y, res_id_up(up[y]), res_id_down(down[y]), zfree};
      } else if (!Pl.empty()) {  // Change: both chains of the same data node
        const int x = Pl[pick(h(p, 1), (uint32_t)Pl.size())];
        const int y = Q[pick(h(p, 2), (uint32_t)Q.size())];
        if (tag[x] != tag[y]) continue;
        const int j1 = node_of(down[x]), j2 = node_of(down[y]);
        if (j1 == j2) continue;
        const int64_t dpj2 = d(p, j2), dqj1 = d(q, j1), dpj1 = d(p, j1), dqj2 = d(q, j2);
        if (dpj2 == INF || dqj1 == INF || dpj1 == INF || dqj2 == INF) continue;
        delta = (obj == ORC_OBJ_SUM) ? (dpj2 + dqj1) - (dpj1 + dqj2) : std::max(dpj2, dqj1) - std::max(dpj1, dqj2);
        pr.kind = 1; pr.x = x; pr.y = y;
        pr.touched = {x, y, res_id_down(down[x]), res_id_down(down[y])};
      } else {
        continue;
      }
      if (delta == 0) continue;
      if (delta > 0 && !((h(p, 3) >> 32) < (uint64_t)ann.get(kacc[p], delta))) continue;
      pr.key = ((uint64_t)(delta + (1ll << 40)) << 22) | (uint64_t)p;
      props.push_back(pr);
    }
    const int64_t nres = (int64_t)Sn_ * I.MC + 2 * (int64_t)K * Mmax;
    std::vector<uint64_t> res((size_t)nres, UINT64_MAX);
    for (const Proposal& pr : props) for (int64_t t : pr.touched) res[t] = std::min(res[t], pr.key);
    for (const Proposal& pr : props) {
      bool win = true;
      for (int64_t t : pr.touched) win = win && res[t] == pr.key;
      if (!win) continue;
      if (pr.kind == 1) {
        const int32_t dx = down[pr.x], dy = down[pr.y];
        down[pr.x] = dy; down[pr.y] = dx;
        set_up_of(dy, pr.x); set_up_of(dx, pr.y);
        kacc[pr.gid] += 1;
      } else if (pr.kind == 2) {
        const int32_t a = up[pr.y], cc = down[pr.y];
        up[pr.z] = a; down[pr.z] = cc; tag[pr.z] = tag[pr.y];
        set_down_of(a, pr.z); set_up_of(cc, pr.z);
        up[pr.y] = NONE; down[pr.y] = NONE;
        kacc[pr.gid] += 1;
      } else if (pr.kind == 3) {
        const int32_t a = up[pr.x];
        up[pr.x] = NONE;
        set_down_of(a, NONE);
        deny[pr.gid] = 0;
      }
      ++changes;
    }
    quiet = changes > 0 ? 0 : quiet + 1;
    round += 1;
    return changes;
  }

  void result(int64_t* F_dec, int64_t* cost_dec, int32_t* dangling) const {
    for (int k = 0; k < K; ++k) {
      int64_t F = 0, C = 0;
      for (int64_t i = 0; i < M[k]; ++i) {
        int32_t p = src_down[(size_t)k * Mmax + i];
        if (p == NONE) continue;
        int64_t cc = d(-1 - k, p / I.MC);
        int guard = 0;
        while (p >= 0 && ++guard <= I.S + 1) {
          const int32_t nx = down[p];
          if (nx == NONE) { cc = -1; break; }
          cc = Rounds::sadd(cc, nx <= -2 ? d(p / I.MC, -1 - dk(nx)) : d(p / I.MC, nx / I.MC));
          p = nx;
        }
        if (cc >= 0 && cc != INF && p <= -2 && dk(p) == k) { F += 1; C += cc; }
      }
      F_dec[k] = F;
      cost_dec[k] = C;
    }
    int32_t dang = 0;
    for (size_t p = 0; p < up.size(); ++p) if (st((int)p) == OUT) ++dang;
    *dangling = dang;
  }

  // digest: per slot (state, enc(up), enc(down), tag + 1 if not FREE else 0); SRC_k / SNK_k in
  // (k, i) order; (kacc, deny) per relay; quiet.  enc: relay slot 1 + p, SRC_k i 2^40 + k 2^20 + i,
  // SNK_k i 2^41 + k 2^20 + i, none 0
  uint64_t digest() const {
    uint64_t dg = 0, pos = 0;
    auto add = [&](uint64_t val) { dg += mix64(mix64(pos) ^ val); ++pos; };
    auto enc = [&](int32_t p, uint64_t side) -> uint64_t {
      return p == NONE ? 0 : p >= 0 ? 1 + (uint64_t)p : side + ((uint64_t)dk(p) << 20) + (uint64_t)di(p);
    };
    for (size_t p = 0; p < up.size(); ++p) {
      const int s = st((int)p);
      add((uint64_t)s); add(enc(up[p], 1ull << 40)); add(enc(down[p], 1ull << 41));
      add(s == FREE ? 0 : (uint64_t)tag[p] + 1);
    }
    for (int k = 0; k < K; ++k)
      for (int64_t i = 0; i < Mmax; ++i) add(src_down[(size_t)k * Mmax + i] == NONE ? 0 : 1 + (uint64_t)src_down[(size_t)k * Mmax + i]);
    for (int k = 0; k < K; ++k)
      for (int64_t i = 0; i < Mmax; ++i) add(snk_up[(size_t)k * Mmax + i] == NONE ? 0 : 1 + (uint64_t)snk_up[(size_t)k * Mmax + i]);
    for (int g = 0; g < Sn(); ++g) { add((uint64_t)(uint32_t)kacc[g]); add((uint64_t)(uint32_t)deny[g]); }
    add((uint64_t)(uint32_t)quiet);
    return dg;
  }
};
struct orc_mc_rounds { McRounds R; };


extern "C" {

int orc_eq1(int32_t S, int32_t n, int32_t L, const int32_t* comp, const int32_t* loc, int32_t dloc,
            const int32_t* lat, const int32_t* bw, int64_t size_kbit, int32_t* src, int32_t* snk, int32_t* link) {
  auto LAT = [&](int a, int b) { return lat[a * L + b]; };
  auto BW = [&](int a, int b) { return bw[a * L + b]; };
  for (int i = 0; i < n; ++i) {
    const int li = loc[i];  // stage 0
    src[i] = (int32_t)eq1_d2(0, comp[i], LAT(dloc, li), LAT(li, dloc), BW(dloc, li), BW(li, dloc), size_kbit);
    const int k = (S - 1) * n + i, lk = loc[k];
    snk[i] = (int32_t)eq1_d2(comp[k], 0, LAT(lk, dloc), LAT(dloc, lk), BW(lk, dloc), BW(dloc, lk), size_kbit);
  }
  for (int s = 0; s + 1 < S; ++s)
    for (int v = 0; v < n; ++v)
      for (int u = 0; u < n; ++u) {
        const int a = s * n + u, b = (s + 1) * n + v;
        link[((size_t)s * n + v) * n + u] =
            (int32_t)eq1_d2(comp[a], comp[b], LAT(loc[a], loc[b]), LAT(loc[b], loc[a]), BW(loc[a], loc[b]),
                            BW(loc[b], loc[a]), size_kbit);
      }
  return 0;
}

int orc_ssp(const orc_instance* Iv, int64_t* F, int64_t* cost, int32_t* A, int32_t* node_flow,
            int32_t* src_flow, int32_t* snk_flow, int32_t* arc_flow, int64_t* cost_curve) {
  Inst I(Iv);
  Flow fl(I);
  std::vector<int64_t> curve;
  const int rc = ssp(I, fl, &curve);
  if (rc) return rc;
  if (F) *F = fl.F;
  if (cost) *cost = fl.cost;
  if (A) *A = fl.A;
  if (node_flow) std::copy(fl.g.begin(), fl.g.end(), node_flow);
  if (src_flow) std::copy(fl.src_f.begin(), fl.src_f.end(), src_flow);
  if (snk_flow) std::copy(fl.snk_f.begin(), fl.snk_f.end(), snk_flow);
  if (arc_flow) std::copy(fl.arc.begin(), fl.arc.end(), arc_flow);
  if (cost_curve) {
    // cost_curve[m] = min cost of a flow of value m, m = 0..F (solve with supply m)
    cost_curve[0] = 0;
    for (int64_t m = 1; m <= fl.F; ++m) {
      orc_instance J = *Iv;
      J.M = m;
      Inst IJ(&J);
      Flow fj(IJ);
      if (ssp(IJ, fj, nullptr)) return -20;
      cost_curve[m] = fj.cost;
    }
  }
  return 0;
}

int orc_ssp_batch(int64_t B, int32_t S, int32_t n, int32_t max_cap, const int32_t* cap, const uint8_t* alive,
                  const int32_t* src, const int32_t* snk, const int32_t* link, const int64_t* supply, int64_t* F,
                  int64_t* cost, int32_t* A, int32_t threads) {
  std::atomic<int> err{0};
  parallel_for(B, threads, [&](int64_t b) {
    orc_instance v = view(b, S, n, max_cap, cap, alive, src, snk, link, supply);
    Inst I(&v);
    Flow fl(I);
    if (ssp(I, fl, nullptr)) err = 1;
    F[b] = fl.F; cost[b] = fl.cost; A[b] = fl.A;
  });
  return err.load() ? -1 : 0;
}

int orc_warm_reroute(const orc_instance* Iold_v, const int32_t* node_flow, const int32_t* src_flow,
                     const int32_t* snk_flow, const int32_t* arc_flow, const orc_instance* Inew_v, int64_t* F,
                     int64_t* cost, int64_t* stats, int32_t* node_flow_out, int32_t* src_flow_out,
                     int32_t* snk_flow_out, int32_t* arc_flow_out) {
  Inst Io(Iold_v), In(Inew_v);
  if (Io.S != In.S || Io.n != In.n) return -30;
  Flow fo(Io), fn(In);
  std::copy(node_flow, node_flow + fo.g.size(), fo.g.begin());
  std::copy(src_flow, src_flow + Io.n, fo.src_f.begin());
  std::copy(snk_flow, snk_flow + Io.n, fo.snk_f.begin());
  if (arc_flow) std::copy(arc_flow, arc_flow + fo.arc.size(), fo.arc.begin());
  WarmStats st;
  const int rc = warm_reroute(Io, fo, In, fn, st);
  if (rc) return rc;
  if (F) *F = fn.F;
  if (cost) *cost = fn.cost;
  if (stats) { stats[0] = st.stripped; stats[1] = st.cycles; stats[2] = st.augment; }
  if (node_flow_out) std::copy(fn.g.begin(), fn.g.end(), node_flow_out);
  if (src_flow_out) std::copy(fn.src_f.begin(), fn.src_f.end(), src_flow_out);
  if (snk_flow_out) std::copy(fn.snk_f.begin(), fn.snk_f.end(), snk_flow_out);
  if (arc_flow_out) std::copy(fn.arc.begin(), fn.arc.end(), arc_flow_out);
  return 0;
}

int orc_network_simplex(const orc_instance* Iv, int64_t* F, int64_t* cost) {
  Inst I(Iv);
  return network_simplex(I, F, cost);
}

int orc_certify(const orc_instance* Iv, int64_t F, int64_t cost, const int32_t* node_flow, const int32_t* src_flow,
                const int32_t* snk_flow, const int32_t* arc_flow) {
  Inst I(Iv);
  Flow fl(I);
  std::copy(node_flow, node_flow + fl.g.size(), fl.g.begin());
  std::copy(src_flow, src_flow + I.n, fl.src_f.begin());
  std::copy(snk_flow, snk_flow + I.n, fl.snk_f.begin());
  std::copy(arc_flow, arc_flow + fl.arc.size(), fl.arc.begin());
  return certify(I, fl, F, cost);
}

int orc_anneal_table(double T0, double alpha, int32_t* width, int32_t* K, uint32_t* table, int64_t cap) {
  Anneal a;
  const int rc = a.init(T0, alpha);
  if (rc) return rc;
  if (width) *width = a.width;
  if (K) *K = a.K;
  if (table) {
    if ((int64_t)a.t.size() > cap) return -5;
    std::copy(a.t.begin(), a.t.end(), table);
  }
  return 0;
}

orc_rounds* orc_rounds_create(const orc_instance* I, uint64_t seed, int64_t inst_id, double T0, double alpha,
                              int32_t objective, int32_t W, int32_t deny_after) {
  if (!I || I->S < 1 || I->n < 1 || I->max_cap < 0 || I->M < 0 || W < 1 || deny_after < 1) return nullptr;
  orc_rounds* o = new orc_rounds();
  o->R.I = Inst(I);
  o->R.seed = seed;
  o->R.inst = inst_id;
  o->R.obj = objective;
  o->R.W = W;
  o->R.deny_after = deny_after;
  if (o->R.ann.init(T0, alpha)) { delete o; return nullptr; }
  o->R.reset_state();
  return o;
}

void orc_rounds_destroy(orc_rounds* R) { delete R; }

int orc_rounds_run(orc_rounds* o, int32_t max_rounds, int32_t* rounds_run, int64_t* F_dec, int64_t* cost_dec,
                   int32_t* dangling, uint64_t* digests) {
  Rounds& R = o->R;
  R.quiet = 0;
  int32_t r = 0;
  while (r < max_rounds) {
    R.one_round();
    if (digests) digests[r] = R.digest();
    ++r;
    if (R.quiet >= R.W) break;
  }
  if (rounds_run) *rounds_run = r;
  int64_t f = 0, c = 0;
  int32_t dg = 0;
  R.result(&f, &c, &dg);
  if (F_dec) *F_dec = f;
  if (cost_dec) *cost_dec = c;
  if (dangling) *dangling = dg;
  return 0;
}

int orc_rounds_apply_churn(orc_rounds* o, const uint8_t* alive_new, const int32_t* updates, int64_t k) {
  o->R.apply_churn(alive_new, updates, updates ? k : 0);
  return 0;
}

int orc_rounds_export(const orc_rounds* o, int32_t* up, int32_t* down, int32_t* src_down, int32_t* snk_up,
                      int32_t* kacc, int32_t* deny, int32_t* quiet, int64_t* round) {
  const Rounds& R = o->R;
  if (up) std::copy(R.up.begin(), R.up.end(), up);
  if (down) std::copy(R.down.begin(), R.down.end(), down);
  if (src_down) std::copy(R.src_down.begin(), R.src_down.end(), src_down);
  if (snk_up) std::copy(R.snk_up.begin(), R.snk_up.end(), snk_up);
  if (kacc) std::copy(R.kacc.begin(), R.kacc.end(), kacc);
  if (deny) std::copy(R.deny.begin(), R.deny.end(), deny);
  if (quiet) *quiet = R.quiet;
  if (round) *round = R.round;
  return 0;
}

// Inverse of orc_rounds_export (checkpoint / resume): the caller supplies a state in the
// export layouts.  Checked here: the pairing bijectivity and capacity invariants,
// pointers only across one stage boundary (or to the data node at the ends); -1 when violated.
int orc_rounds_import(orc_rounds* o, const int32_t* up, const int32_t* down, const int32_t* src_down,
                      const int32_t* snk_up, const int32_t* kacc, const int32_t* deny, int32_t quiet, int64_t round) {
  Rounds& R = o->R;
  const Inst& I = R.I;
  const int S = I.S, n = I.n, MC = I.MC;
  const int64_t ns = (int64_t)S * n * MC, M = I.M;
  for (int64_t p = 0; p < ns; ++p) {
    const int g = (int)(p / MC), j = (int)(p % MC), s = g / n;
    const bool usable = R.alive(g) && j < R.capE(g);
    if (!usable && (up[p] != NONE || down[p] != NONE)) return -1;
    if (up[p] >= 0 && (up[p] >= ns || up[p] / MC / n != s - 1 || down[up[p]] != (int32_t)p)) return -1;
    if (up[p] <= -2 && (s != 0 || -2 - up[p] >= M || src_down[-2 - up[p]] != (int32_t)p)) return -1;
    if (down[p] >= 0 && (down[p] >= ns || down[p] / MC / n != s + 1 || up[down[p]] != (int32_t)p)) return -1;
    if (down[p] <= -2 && (s != S - 1 || -2 - down[p] >= M || snk_up[-2 - down[p]] != (int32_t)p)) return -1;
  }
  for (int64_t k = 0; k < M; ++k) {
    if (src_down[k] != NONE && (src_down[k] < 0 || src_down[k] >= ns || up[src_down[k]] != (int32_t)(-2 - k))) return -1;
    if (snk_up[k] != NONE && (snk_up[k] < 0 || snk_up[k] >= ns || down[snk_up[k]] != (int32_t)(-2 - k))) return -1;
  }
  R.up.assign(up, up + ns);
  R.down.assign(down, down + ns);
  R.src_down.assign(src_down, src_down + M);
  R.snk_up.assign(snk_up, snk_up + M);
  R.kacc.assign(kacc, kacc + (size_t)S * n);
  R.deny.assign(deny, deny + (size_t)S * n);
  R.quiet = quiet;
  R.round = round;
  return 0;
}

// The counter-based draws of R4: h(gid, stream) of an instance/round, and
// pick(x, m) = floor((x >> 32) * m / 2^32); exported for the known-answer tests.
uint64_t orc_mix64(uint64_t z) { return mix64(z); }
uint64_t orc_rng_h(uint64_t seed, int64_t inst, int64_t round, int32_t gid, int32_t stream) {
  Rounds R;
  R.seed = seed;
  R.inst = inst;
  R.round = round;
  return R.h(gid, stream);
}
uint32_t orc_pick(uint64_t x, uint32_t m) { return pick(x, m); }

uint64_t orc_rounds_digest(const orc_rounds* o) { return o->R.digest(); }

int orc_rounds_instance(const orc_rounds* o, int32_t* cap_eff, uint8_t* alive, int32_t* src, int32_t* snk,
                        int32_t* link) {
  const Inst& I = o->R.I;
  if (cap_eff) for (int s = 0; s < I.S; ++s) for (int i = 0; i < I.n; ++i) cap_eff[s * I.n + i] = I.capE(s, i);
  if (alive) std::copy(I.alive.begin(), I.alive.end(), alive);
  if (src) std::copy(I.src.begin(), I.src.end(), src);
  if (snk) std::copy(I.snk.begin(), I.snk.end(), snk);
  if (link) std::copy(I.link.begin(), I.link.end(), link);
  return 0;
}

int32_t orc_llama_victim(const orc_rounds* o, uint64_t draw_stage, uint64_t draw_pick) {
  const Rounds& R = o->R;
  const int S = R.I.S, n = R.I.n;
  const int s0 = (int)pick(draw_stage, (uint32_t)S);
  for (int t = 0; t < S; ++t) {
    const int s = (s0 + t) % S;
    std::vector<int> cand;
    for (int i = 0; i < n; ++i) {
      const int g = s * n + i;
      bool paired = false;
      for (int j = 0; j < R.capE(g); ++j) paired = paired || R.st(R.slot(g, j)) == PAIRED;
      if (R.alive(g) && paired) cand.push_back(g);
    }
    if (!cand.empty()) return cand[pick(draw_pick, (uint32_t)cand.size())];
  }
  return -1;
}

int orc_pipeline_batch(int64_t B, int32_t S, int32_t n, int32_t max_cap, const int32_t* cap, const uint8_t* alive,
                       const int32_t* src, const int32_t* snk, const int32_t* link, const int64_t* supply,
                       int32_t churn_kind, const uint8_t* alive_new, const int32_t* updates, int64_t k_updates,
                       const uint64_t* victim_draws, uint64_t seed, int64_t inst_base, double T0, double alpha,
                       int32_t objective, int32_t W, int32_t deny_after, int32_t max_rounds, int32_t threads,
                       orc_result* out) {
  // updates are sorted by instance (column 0 = local instance index); find each instance's range
  std::vector<int64_t> ubeg(B + 1, 0);
  if (updates && k_updates > 0) {
    for (int64_t e = 0; e < k_updates; ++e) {
      const int64_t b = updates[5 * e];
      if (b < 0 || b >= B) return -2;
      ubeg[b + 1] += 1;
    }
    for (int64_t b = 0; b < B; ++b) ubeg[b + 1] += ubeg[b];
    for (int64_t e = 1; e < k_updates; ++e) if (updates[5 * e] < updates[5 * (e - 1)]) return -3;
  }
  std::atomic<int> err{0};
  parallel_for(B, threads, [&](int64_t b) {
    orc_instance v = view(b, S, n, max_cap, cap, alive, src, snk, link, supply);
    orc_rounds* R = orc_rounds_create(&v, seed, inst_base + b, T0, alpha, objective, W, deny_after);
    if (!R) { err = 1; return; }
    orc_result& r = out[b];
    int64_t fd, cd;
    int32_t dg, pre = 0;
    orc_rounds_run(R, max_rounds, &pre, &fd, &cd, &dg, nullptr);
    // the bench step's work starts here (the pre-churn rounds are its untimed setup)
    const auto t_step = std::chrono::steady_clock::now();
    if (churn_kind == 1) {
      orc_rounds_apply_churn(R, alive_new ? alive_new + b * S * n : nullptr,
                             updates ? updates + 5 * ubeg[b] : nullptr, ubeg[b + 1] - ubeg[b]);
    } else if (churn_kind == 2) {
      const int32_t vic = orc_llama_victim(R, victim_draws[2 * b], victim_draws[2 * b + 1]);
      std::vector<uint8_t> al(R->R.I.alive);
      if (vic >= 0) al[vic] = 0;
      orc_rounds_apply_churn(R, al.data(), nullptr, 0);
    }
    // cold SSP on the masked graph
    const Inst& M = R->R.I;
    Flow fl(M);
    if (ssp(M, fl, nullptr)) err = 2;
    r.F = fl.F; r.cost = fl.cost; r.A = fl.A;
    int32_t rr = 0;
    orc_rounds_run(R, max_rounds, &rr, &r.F_dec, &r.cost_dec, &r.dangling, nullptr);
    r.rounds = rr;
    r.pre_rounds = pre;
    r.step_ns = (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_step).count();
    r.digest = orc_rounds_digest(R);
    orc_rounds_destroy(R);
  });
  return err.load() ? -1 : 0;
}

// ---- multi-data-node rounds (MC-SYNC) ----
orc_mc_rounds* orc_mc_rounds_create(const orc_instance* I, int32_t K, const int32_t* src_k, const int32_t* snk_k,
                                    const int64_t* M_k, uint64_t seed, int64_t inst_id, double T0, double alpha,
                                    int32_t objective, int32_t W, int32_t deny_after) {
  if (!I || K < 1 || I->S < 1 || I->n < 1 || W < 1 || deny_after < 1) return nullptr;
  orc_mc_rounds* o = new orc_mc_rounds();
  McRounds& R = o->R;
  R.I = Inst(I);
  R.K = K;
  R.M.assign(M_k, M_k + K);
  R.Mmax = 1;
  for (int k = 0; k < K; ++k) R.Mmax = std::max<int64_t>(R.Mmax, R.M[k]);
  R.srcK.assign(src_k, src_k + (size_t)K * I->n);
  R.snkK.assign(snk_k, snk_k + (size_t)K * I->n);
  R.seed = seed; R.inst = inst_id; R.obj = objective; R.W = W; R.deny_after = deny_after;
  if (R.ann.init(T0, alpha)) { delete o; return nullptr; }
  R.reset_state();
  return o;
}
void orc_mc_rounds_destroy(orc_mc_rounds* o) { delete o; }
int orc_mc_rounds_run(orc_mc_rounds* o, int32_t max_rounds, int32_t* rounds_run, int64_t* F_dec, int64_t* cost_dec,
                      int32_t* dangling, uint64_t* digests) {
  McRounds& R = o->R;
  R.quiet = 0;
  int32_t r = 0;
  while (r < max_rounds) {
    R.one_round();
    if (digests) digests[r] = R.digest();
    ++r;
    if (R.quiet >= R.W) break;
  }
  if (rounds_run) *rounds_run = r;
  std::vector<int64_t> f(R.K), c(R.K);
  int32_t dg = 0;
  R.result(f.data(), c.data(), &dg);
  for (int k = 0; k < R.K; ++k) { if (F_dec) F_dec[k] = f[k]; if (cost_dec) cost_dec[k] = c[k]; }
  if (dangling) *dangling = dg;
  return 0;
}
int orc_mc_rounds_export(const orc_mc_rounds* o, int32_t* up, int32_t* down, int32_t* tag, int32_t* src_down,
                         int32_t* snk_up, int32_t* kacc, int32_t* deny, int32_t* quiet, int64_t* round) {
  const McRounds& R = o->R;
  if (up) std::copy(R.up.begin(), R.up.end(), up);
  if (down) std::copy(R.down.begin(), R.down.end(), down);
  if (tag) for (size_t p = 0; p < R.tag.size(); ++p) tag[p] = R.st((int)p) == FREE ? -1 : R.tag[p];
  if (src_down) std::copy(R.src_down.begin(), R.src_down.end(), src_down);
  if (snk_up) std::copy(R.snk_up.begin(), R.snk_up.end(), snk_up);
  if (kacc) std::copy(R.kacc.begin(), R.kacc.end(), kacc);
  if (deny) std::copy(R.deny.begin(), R.deny.end(), deny);
  if (quiet) *quiet = R.quiet;
  if (round) *round = R.round;
  return 0;
}
uint64_t orc_mc_rounds_digest(const orc_mc_rounds* o) { return o->R.digest(); }

// Install an MC round state in the export layouts (tag -1 on FREE slots); kacc / deny / quiet may be
// NULL (0).  -1 (state unchanged) unless it is a valid pairing whose pointers cross one stage
// boundary, whose data-node slots are below their supply, and whose every link joins slots of one tag,
// SRC_k / SNK_k only slots tagged k.
int orc_mc_rounds_import(orc_mc_rounds* o, const int32_t* up, const int32_t* down, const int32_t* tag,
                         const int32_t* src_down, const int32_t* snk_up, const int32_t* kacc, const int32_t* deny,
                         int32_t quiet, int64_t round) {
  McRounds& R = o->R;
  const Inst& I = R.I;
  const int S = I.S, n = I.n, MC = I.MC, K = R.K;
  const int64_t ns = (int64_t)S * n * MC, Mm = R.Mmax;
  auto dk = [&](int32_t p) { return (int)((-2 - (int64_t)p) / Mm); };
  auto di = [&](int32_t p) { return (-2 - (int64_t)p) % Mm; };
  for (int64_t p = 0; p < ns; ++p) {
    const int g = (int)(p / MC), j = (int)(p % MC), s = g / n;
    const bool usable = R.alive(g) && j < R.capE(g);
    const bool free_ = up[p] == NONE && down[p] == NONE;
    if (!usable && !free_) return -1;
    if (!free_ && (tag[p] < 0 || tag[p] >= K)) return -1;
    if (up[p] >= 0 && (up[p] >= ns || up[p] / MC / n != s - 1 || down[up[p]] != (int32_t)p || tag[up[p]] != tag[p])) return -1;
    if (up[p] <= -2 && (s != 0 || dk(up[p]) >= K || dk(up[p]) != tag[p] || di(up[p]) >= R.M[dk(up[p])] ||
                        src_down[(size_t)dk(up[p]) * Mm + di(up[p])] != (int32_t)p)) return -1;
    if (down[p] >= 0 && (down[p] >= ns || down[p] / MC / n != s + 1 || up[down[p]] != (int32_t)p || tag[down[p]] != tag[p])) return -1;
    if (down[p] <= -2 && (s != S - 1 || dk(down[p]) >= K || dk(down[p]) != tag[p] || di(down[p]) >= R.M[dk(down[p])] ||
                          snk_up[(size_t)dk(down[p]) * Mm + di(down[p])] != (int32_t)p)) return -1;
  }
  for (int k = 0; k < K; ++k)
    for (int64_t i = 0; i < Mm; ++i) {
      const int32_t sd = src_down[(size_t)k * Mm + i], su = snk_up[(size_t)k * Mm + i];
      if (i >= R.M[k] && (sd != NONE || su != NONE)) return -1;
      if (sd != NONE && (sd < 0 || sd >= ns || up[sd] != McRounds::dptr(k, i, Mm))) return -1;
      if (su != NONE && (su < 0 || su >= ns || down[su] != McRounds::dptr(k, i, Mm))) return -1;
    }
  R.up.assign(up, up + ns);
  R.down.assign(down, down + ns);
  for (int64_t p = 0; p < ns; ++p) R.tag[p] = tag[p] < 0 ? 0 : tag[p];
  R.src_down.assign(src_down, src_down + (size_t)K * Mm);
  R.snk_up.assign(snk_up, snk_up + (size_t)K * Mm);
  if (kacc) R.kacc.assign(kacc, kacc + (size_t)S * n); else R.kacc.assign((size_t)S * n, 0);
  if (deny) R.deny.assign(deny, deny + (size_t)S * n); else R.deny.assign((size_t)S * n, 0);
  R.quiet = quiet;
  R.round = round;
  return 0;
}

}  // extern "C"
