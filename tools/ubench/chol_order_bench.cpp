#include <vector>
#include <queue>
#include <algorithm>
#include <iterator>
#include <numeric>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <chrono>
using clk = std::chrono::steady_clock;
double ms_since(clk::time_point t){ return std::chrono::duration<double,std::milli>(clk::now()-t).count(); }
constexpr int PART_MIN = 12, PART_CHUNK = 8;
void min_degree_lists(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                      std::vector<std::vector<int>>& colstruct);

// Same elimination (repeatedly the live node of smallest (degree, id); its live
// neighbours become a clique) on adjacency bitsets: a neighbour update is W word
// ORs instead of a sorted-list merge.  Identical order and column structures to
// min_degree_lists; used while the core fits in a few hundred words per row.
void min_degree(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                std::vector<std::vector<int>>& colstruct) {
  const int W = (m + 63) / 64;
  if (m > 8192) {
    min_degree_lists(m, adj, order, colstruct);
    return;
  }
  order.clear();
  order.reserve(m);
  colstruct.assign(m, {});
  std::vector<uint64_t> bits((size_t)m * W, 0ull), nb(W);
  std::vector<int> deg(m);
  for (int v = 0; v < m; ++v) {
    uint64_t* r = bits.data() + (size_t)v * W;
    for (int a : adj[v]) r[a >> 6] |= 1ull << (a & 63);
    deg[v] = (int)adj[v].size();
  }
  std::vector<char> done(m, 0);
  typedef std::pair<int, int> DI;
  std::vector<DI> hv;
  hv.reserve(2 * m);
  for (int v = 0; v < m; ++v) hv.push_back({deg[v], v});
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap(std::greater<DI>(), std::move(hv));
  std::vector<int> list;
  while (!heap.empty()) {
    DI top = heap.top();
    heap.pop();
    const int v = top.second;
    if (done[v] || top.first != deg[v]) continue;
    done[v] = 1;
    order.push_back(v);
    const uint64_t* rv = bits.data() + (size_t)v * W;
    std::copy(rv, rv + W, nb.begin());
    list.clear();
    for (int w = 0; w < W; ++w)
      for (uint64_t x = nb[w]; x; x &= x - 1) list.push_back(64 * w + __builtin_ctzll(x));
    colstruct[v] = list;  // ascending ids, as the sorted lists
    for (int a : list) {
      uint64_t* ra = bits.data() + (size_t)a * W;
      int d = 0;
      for (int w = 0; w < W; ++w) {
        ra[w] |= nb[w];
        if (w == (a >> 6)) ra[w] &= ~(1ull << (a & 63));
        if (w == (v >> 6)) ra[w] &= ~(1ull << (v & 63));
        d += __builtin_popcountll(ra[w]);
      }
      deg[a] = d;
      heap.push({d, a});
    }
  }
}

void min_degree_lists(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                      std::vector<std::vector<int>>& colstruct) {
  order.clear();
  order.reserve(m);
  colstruct.assign(m, {});
  std::vector<char> done(m, 0);
  typedef std::pair<int, int> DI;
  std::vector<DI> hv;
  hv.reserve(2 * m);
  for (int v = 0; v < m; ++v) hv.push_back({(int)adj[v].size(), v});
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap(std::greater<DI>(), std::move(hv));
  std::vector<int> merged;
  while (!heap.empty()) {
    DI top = heap.top();
    heap.pop();
    int v = top.second;
    if (done[v] || top.first != (int)adj[v].size()) continue;
    done[v] = 1;
    order.push_back(v);
    std::vector<int>& nb = colstruct[v];
    nb.swap(adj[v]);
    for (int a : nb) {
      merged.clear();
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      std::vector<int>& out = adj[a];
      out.clear();
      for (int u : merged)
        if (u != a && u != v) out.push_back(u);
      heap.push({(int)out.size(), a});
    }
  }
}

constexpr double ORDER_REUSE_FILL = 1.05;  // factor blocks and update pairs, over the fresh order's

// Symbolic factorization of the local graph (adjacency adj_ptr / adj_idx, full
// degrees deg) under the cached global elimination order `gorder`, preceded by the
// nodes not in it (ascending local id).  Column structure of v = its later
// neighbours plus its elimination-tree children's structures minus v, sorted by
// position.  Fills order / pos / csp / csi as the fresh ordering does; false when the
// factor would exceed max_nnz off-diagonal blocks or max_upd update pairs.
bool symbolic_fixed_order(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj_idx,
                          const std::vector<int>& deg, const std::vector<int>& loc, const std::vector<int>& gorder,
                          int64_t max_nnz, int64_t max_upd, std::vector<int>* scratch, std::vector<int>& order,
                          std::vector<int>& pos, std::vector<int>& csp, std::vector<int>& csi) {
  int64_t upd = 0;
  std::vector<int>&seen = scratch[0], &mark = scratch[1], &head = scratch[2], &nxt = scratch[3], &st0 = scratch[4],
                  &len = scratch[5], &flat = scratch[6], &L = scratch[7];
  seen.assign(m, 0);
  order.clear();
  for (int g : gorder)
    if (loc[g] >= 0) seen[loc[g]] = 1;
  for (int v = 0; v < m; ++v)
    if (!seen[v]) order.push_back(v);
  for (int g : gorder)
    if (loc[g] >= 0) order.push_back(loc[g]);
  if ((int)order.size() != m) return false;
  pos.resize(m);
  for (int i = 0; i < m; ++i) pos[order[i]] = i;
  mark.assign(m, -1);
  head.assign(m, -1);
  nxt.assign(m, -1);
  st0.assign(m, 0);
  len.assign(m, 0);
  flat.clear();
  for (int i = 0; i < m; ++i) {
    const int v = order[i];
    L.clear();
    for (int e = adj_ptr[v]; e < adj_ptr[v] + deg[v]; ++e) {
      const int u = adj_idx[e];
      if (pos[u] > i && mark[u] != v) {
        mark[u] = v;
        L.push_back(u);
      }
    }
    for (int c = head[v]; c >= 0; c = nxt[c])
      for (int k = st0[c]; k < st0[c] + len[c]; ++k) {
        const int u = flat[k];
        if (u != v && mark[u] != v) {
          mark[u] = v;
          L.push_back(u);
        }
      }
    std::sort(L.begin(), L.end(), [&](int a, int b) { return pos[a] < pos[b]; });
    st0[v] = (int)flat.size();
    len[v] = (int)L.size();
    flat.insert(flat.end(), L.begin(), L.end());
    upd += (int64_t)L.size() * ((int64_t)L.size() - 1) / 2;  // update pairs of this column
    if ((int64_t)flat.size() > max_nnz || upd > max_upd) return false;
    if (!L.empty()) {
      nxt[v] = head[L[0]];
      head[L[0]] = v;
    }
  }
  csp.assign(m + 1, 0);
  for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + len[v];
  csi.resize(csp[m]);
  for (int v = 0; v < m; ++v) std::copy(flat.begin() + st0[v], flat.begin() + st0[v] + len[v], csi.begin() + csp[v]);
  return true;
}


struct An { int n_cta=0; int64_t n_edges=0; int n_coupled=0; int64_t n_blk=0, n_upd=0; int max_level=0, largest=0; double ms_order=0, ms_sub[6]={}; bool order_reused=false;};
struct CC { bool valid=false; int n=0; std::vector<int> gorder; int64_t fresh_nnz=0, fresh_upd=0; };
struct Wk { std::vector<int> hs_i[40]; std::vector<char> hs_c[4]; CC ch_cache; };
void run(int n, std::vector<uint64_t>& cur, Wk& w, An& an){
  auto t0 = clk::now();
  CC& cc = w.ch_cache;
  // coupled nodes (>= 1 nonzero coupling) get local ids in ascending node order;
  // host scratch persists across analyses (no allocations in the steady state)
  std::vector<int>&loc = w.hs_i[0], &glob = w.hs_i[1], &adj_ptr = w.hs_i[2], &adj_idx = w.hs_i[3],
                  &deg = w.hs_i[4], &live = w.hs_i[5], &live2 = w.hs_i[6], &sel = w.hs_i[7], &cs0 = w.hs_i[8],
                  &cs1 = w.hs_i[9], &order = w.hs_i[10], &pos = w.hs_i[11], &csp = w.hs_i[12], &csi = w.hs_i[13];
  std::vector<char>&gone = w.hs_c[0], &blocked = w.hs_c[1];
  const double ms_cur = ms_since(t0);
  loc.assign(n, -1);
  glob.clear();
  for (uint64_t e : cur) {
    loc[(int)(e >> 32)] = 0;
    loc[(int)(e & 0xffffffffu)] = 0;
    ++an.n_edges;
  }
  for (int v = 0; v < n; ++v)
    if (loc[v] == 0) {
      loc[v] = (int)glob.size();
      glob.push_back(v);
    }
  const int m = (int)glob.size();
  an.n_coupled = m;
  adj_ptr.assign(m + 1, 0);
  adj_idx.resize(2 * an.n_edges);
  for (uint64_t e : cur) {
    adj_ptr[loc[(int)(e >> 32)] + 1]++;
    adj_ptr[loc[(int)(e & 0xffffffffu)] + 1]++;
  }
  for (int v = 0; v < m; ++v) adj_ptr[v + 1] += adj_ptr[v];
  deg.assign(m, 0);
  for (uint64_t e : cur) {
    const int a2 = loc[(int)(e >> 32)], b2 = loc[(int)(e & 0xffffffffu)];
    adj_idx[adj_ptr[a2] + deg[a2]++] = b2;
    adj_idx[adj_ptr[b2] + deg[b2]++] = a2;
  }
  const double ms_adj = ms_since(t0);
  // Order reuse: a miss inside a step (the union graph grew by a few contacts)
  // keeps the step's fresh elimination order -- nodes new to the graph first -- and
  // redoes only the symbolic factorization, unless the fill grows by more than
  // ORDER_REUSE_FILL over the fresh order's, in factor blocks or update pairs (then
  // the graph is ordered afresh).
  static const bool no_reuse = getenv("ABD_CHOL_NO_ORDER_REUSE") != nullptr;
  int n_core = 0;
  bool reused = false;
  if (!no_reuse && cc.valid && cc.n == n && !cc.gorder.empty())
    reused = symbolic_fixed_order(m, adj_ptr, adj_idx, deg, loc, cc.gorder, (int64_t)(ORDER_REUSE_FILL * cc.fresh_nnz),
                                  (int64_t)(ORDER_REUSE_FILL * cc.fresh_upd), w.hs_i + 31, order, pos, csp, csi);
  if (!reused) {
    // Elimination order by tree contraction (contact graphs of piles are forests of
    // stacked chains): rounds of rake (every node of degree <= 1 at the start of the
    // round; no fill) and compress (an independent set of degree-2 nodes; the fill
    // edge joins the two neighbours), so a chain of L bodies is eliminated in
    // O(log L) elimination-tree levels instead of L / 2.  What remains (degree >= 3
    // everywhere) is ordered by minimum degree.  cs0/cs1 = the live neighbours of a
    // raked / compressed node when it is eliminated (its L column structure).
    // The live neighbour list of v is adj_idx[adj_ptr[v], adj_ptr[v] + deg[v]),
    // edited in place: rake and compress never raise a degree.
    order.clear();
    cs0.assign(m, -1);
    cs1.assign(m, -1);
    gone.assign(m, 0);
    blocked.assign(m, 0);
    live.resize(m);
    std::iota(live.begin(), live.end(), 0);
    static const bool no_compress = getenv("ABD_CHOL_NO_COMPRESS") != nullptr;
    auto drop = [&](int u, int x) {
      int* l = adj_idx.data() + adj_ptr[u];
      const int d = deg[u];
      for (int i = 0; i < d; ++i)
        if (l[i] == x) {
          l[i] = l[d - 1];
          deg[u] = d - 1;
          return;
        }
    };
    auto relink = [&](int u, int x, int y) {  // in u's list: x -> y, or drop x when y is already there
      int* l = adj_idx.data() + adj_ptr[u];
      const int d = deg[u];
      int ix = -1;
      bool has_y = false;
      for (int i = 0; i < d; ++i) {
        if (l[i] == x) ix = i;
        if (l[i] == y) has_y = true;
      }
      if (has_y) {
        l[ix] = l[d - 1];
        deg[u] = d - 1;
      } else {
        l[ix] = y;
      }
    };
    for (;;) {
      bool progress = false;
      sel.clear();
      for (int v : live)
        if (deg[v] <= 1) sel.push_back(v);
      for (int v : sel) {  // rake (a lone pair: the second end follows with no neighbour)
        if (gone[v]) continue;
        if (deg[v] == 1) {
          const int u = adj_idx[adj_ptr[v]];
          cs0[v] = u;
          drop(u, v);
        }
        deg[v] = 0;
        gone[v] = 1;
        order.push_back(v);
        progress = true;
      }
      if (!no_compress) {
        sel.clear();
        for (int v : live) blocked[v] = 0;
        for (int v : live)
          if (!gone[v] && !blocked[v] && deg[v] == 2) {
            const int* l = adj_idx.data() + adj_ptr[v];
            sel.push_back(v);
            blocked[v] = 1;
            blocked[l[0]] = 1;
            blocked[l[1]] = 1;
          }
        for (int v : sel) {  // compress: v's neighbours a, b become adjacent (fill)
          const int* l = adj_idx.data() + adj_ptr[v];
          const int a2 = l[0], b2 = l[1];
          cs0[v] = a2;
          cs1[v] = b2;
          relink(a2, v, b2);
          relink(b2, v, a2);
          deg[v] = 0;
          gone[v] = 1;
          order.push_back(v);
          progress = true;
        }
      }
      live2.clear();
      for (int v : live)
        if (!gone[v]) live2.push_back(v);
      live.swap(live2);
      if (!progress || live.empty()) break;
    }
    const double ms_contract = ms_since(t0);
    n_core = m - (int)order.size();
    std::vector<std::vector<int>> core_cs;
    std::vector<int> core_glob;
    if ((int)order.size() < m) {
      std::vector<int> core_id(m, -1);
      core_glob = live;
      const int mc = (int)core_glob.size();
      for (int c = 0; c < mc; ++c) core_id[core_glob[c]] = c;
      std::vector<std::vector<int>> cadj(mc);
      for (int c = 0; c < mc; ++c) {
        const int v = core_glob[c];
        for (int i = 0; i < deg[v]; ++i) cadj[c].push_back(core_id[adj_idx[adj_ptr[v] + i]]);
        std::sort(cadj[c].begin(), cadj[c].end());
      }
      std::vector<int> corder;
      min_degree(mc, cadj, corder, core_cs);
      for (int c : corder) order.push_back(core_glob[c]);
      for (auto& l : core_cs)
        for (int& x : l) x = core_glob[x];
    }
    const double ms_core = ms_since(t0);
    static const bool trace_ord = getenv("ABD_TRACE_CHOL") != nullptr;
    if (trace_ord)
      fprintf(stderr, "[abd chol order] m=%d core=%d cur_ms=%.3f adj_ms=%.3f contract_ms=%.3f core_ms=%.3f\n", m, n_core,
              ms_cur, ms_adj, ms_contract, ms_core);
    pos.resize(m);
    for (int i = 0; i < m; ++i) pos[order[i]] = i;
    csp.assign(m + 1, 0);
    for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + (cs0[v] >= 0) + (cs1[v] >= 0);
    for (size_t c = 0; c < core_glob.size(); ++c) csp[core_glob[c] + 1] = (int)core_cs[c].size();
    if (!core_glob.empty()) {  // recount: core nodes carry their min-degree column structures
      std::vector<int> cnt(m, 0);
      for (int v = 0; v < m; ++v) cnt[v] = (cs0[v] >= 0) + (cs1[v] >= 0);
      for (size_t c = 0; c < core_glob.size(); ++c) cnt[core_glob[c]] = (int)core_cs[c].size();
      csp[0] = 0;
      for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + cnt[v];
    }
    csi.resize(csp[m]);
    for (int v = 0; v < m; ++v) {
      int* o = csi.data() + csp[v];
      const int k = csp[v + 1] - csp[v];
      if (k == 1) {
        o[0] = cs0[v];
      } else if (k == 2 && cs1[v] >= 0) {
        const bool sw = pos[cs1[v]] < pos[cs0[v]];
        o[0] = sw ? cs1[v] : cs0[v];
        o[1] = sw ? cs0[v] : cs1[v];
      }
    }
    for (size_t c = 0; c < core_glob.size(); ++c) {
      std::vector<int>& l = core_cs[c];
      std::sort(l.begin(), l.end(), [&](int a2, int b2) { return pos[a2] < pos[b2]; });
      std::copy(l.begin(), l.end(), csi.begin() + csp[core_glob[c]]);
    }
    cc.gorder.resize(m);
    for (int i = 0; i < m; ++i) cc.gorder[i] = glob[order[i]];
    cc.fresh_nnz = csp[m];
    cc.fresh_upd = 0;
    for (int v = 0; v < m; ++v) {
      const int64_t k = csp[v + 1] - csp[v];
      cc.fresh_upd += k * (k - 1) / 2;
    }
  }
  an.order_reused = reused;
  an.ms_order = ms_since(t0);
  t0 = clk::now();

  // off-diagonal L blocks: column (local) v owns [col_off[v], col_off[v+1])
  const std::vector<int>& col_off = csp;
  const int nbo = csp[m];
  an.n_blk = n + (int64_t)nbo;
  an.ms_sub[0] = ms_since(t0);
  // row lists (local i): (k, off block) for k eliminated before i, in elimination order of k
  std::vector<int>&rcnt = w.hs_i[14], &rfill = w.hs_i[15], &r_k = w.hs_i[16], &r_b = w.hs_i[17],
                   &upd_ptr = w.hs_i[18], &upd = w.hs_i[19], &level = w.hs_i[20], &root = w.hs_i[21],
                   &csize = w.hs_i[22], &cdepth = w.hs_i[23], &comps = w.hs_i[24];
  rcnt.assign(m + 1, 0);
  for (int e = 0; e < nbo; ++e) rcnt[csi[e] + 1]++;
  for (int v = 0; v < m; ++v) rcnt[v + 1] += rcnt[v];
  rfill.assign(rcnt.begin(), rcnt.end() - 1);
  r_k.resize(nbo);
  r_b.resize(nbo);
  for (int k : order)
    for (int e = csp[k]; e < csp[k + 1]; ++e) {
      int i = csi[e];
      r_k[rfill[i]] = k;
      r_b[rfill[i]] = e;
      rfill[i]++;
    }
  an.ms_sub[1] = ms_since(t0);
  // update pairs for off block (i, j): k in rows(j) with i in cs[k], in elimination
  // order of k.  Every pair (j, i) of cs[k] (j before i) is one such update, so the
  // lists are built by walking each column's pairs once: O(#updates + sum |cs[j]|).
  upd_ptr.assign(nbo + 1, 0);
  std::vector<int>& ub = w.hs_i[29];
  ub.clear();
  // the later entries of cs[k] after j = csi[a2] are a subset of cs[j], both sorted by
  // elimination position: one merge walk finds their blocks in column j
  ub.reserve(4096);
  for (int k : order)
    for (int a2 = csp[k]; a2 < csp[k + 1]; ++a2) {
      const int j = csi[a2];
      int f = csp[j];
      for (int b2 = a2 + 1; b2 < csp[k + 1]; ++b2) {
        const int i = csi[b2];
        while (csi[f] != i) ++f;  // present by the fill property (f < csp[j + 1])
        ub.push_back(f);
        upd_ptr[f + 1]++;
      }
    }
  for (int b = 0; b < nbo; ++b) upd_ptr[b + 1] += upd_ptr[b];
  upd.resize(2 * (size_t)upd_ptr[nbo]);
  {
    std::vector<int>& fill = w.hs_i[30];
    fill.assign(upd_ptr.begin(), upd_ptr.end() - 1);
    size_t q = 0;
    for (int k : order)
      for (int a2 = csp[k]; a2 < csp[k + 1]; ++a2)
        for (int b2 = a2 + 1; b2 < csp[k + 1]; ++b2) {
          const int at = fill[ub[q++]]++;
          upd[2 * (size_t)at] = n + b2;      // L_ik
          upd[2 * (size_t)at + 1] = n + a2;  // L_jk
        }
  }
  an.n_upd = (int64_t)upd.size() / 2;
  an.ms_sub[2] = ms_since(t0);
  // elimination-tree levels and component roots (local)
  level.assign(m, 0);
  root.resize(m);
  for (int v : order)
    if (csp[v + 1] > csp[v]) level[csi[csp[v]]] = std::max(level[csi[csp[v]]], level[v] + 1);
  for (int q = m - 1; q >= 0; --q) {
    int v = order[q];
    root[v] = csp[v + 1] == csp[v] ? v : root[csi[csp[v]]];
  }
  csize.assign(m, 0);
  cdepth.assign(m, 0);
  comps.clear();
  for (int v = 0; v < m; ++v) {
    csize[root[v]]++;
    cdepth[root[v]] = std::max(cdepth[root[v]], level[v] + 1);
    an.max_level = std::max(an.max_level, level[v] + 1);
  }
  for (int v = 0; v < m; ++v)
    if (root[v] == v) comps.push_back(v);
  std::sort(comps.begin(), comps.end(),
            [&](int a, int b) { return csize[a] != csize[b] ? csize[a] > csize[b] : a < b; });
  an.largest = comps.empty() ? 0 : csize[comps[0]];
  static const bool trace_lv = getenv("ABD_TRACE_CHOL") != nullptr;
  if (trace_lv && !comps.empty()) {
    std::vector<int> h(cdepth[comps[0]], 0);
    for (int v = 0; v < m; ++v)
      if (root[v] == comps[0]) h[level[v]]++;
    fprintf(stderr, "[abd chol] largest component levels:");
    for (int x : h) fprintf(stderr, " %d", x);
    fprintf(stderr, "\n");
  }
  an.ms_sub[3] = ms_since(t0);
  an.ms_sub[4] = ms_since(t0);
  // task graph: elimination-tree parents, child lists, leaves (deepest first), isolated nodes
  std::vector<int>&par = w.hs_i[26], &dep = w.hs_i[27], &leaves = w.hs_i[28];
  par.assign(m, -1);
  for (int v = 0; v < m; ++v)
    if (csp[v + 1] > csp[v]) par[v] = csi[csp[v]];
  dep.assign(m, 0);
  for (int q = m - 1; q >= 0; --q) {
    const int v = order[q];
    dep[v] = par[v] < 0 ? 0 : dep[par[v]] + 1;
  }
  std::vector<int> nch(m, 0);
  for (int v = 0; v < m; ++v)
    if (par[v] >= 0) nch[par[v]]++;
  leaves.clear();
  for (int v = 0; v < m; ++v)
    if (nch[v] == 0) leaves.push_back(v);
  std::sort(leaves.begin(), leaves.end(),
            [&](int a2, int b2) { return dep[a2] != dep[b2] ? dep[a2] > dep[b2] : glob[a2] < glob[b2]; });
  const int n_leaves = (int)leaves.size();
  const int n_iso = n - m;
  an.n_cta = 0;  // set at launch
  static const bool trace_cp = getenv("ABD_TRACE_CHOL") != nullptr;
  if (trace_cp) {  // task costs in 12x12 block products: rows + sum over column blocks (1 + updates)
    std::vector<int64_t> cost(m, 0), cp(m, 0);
    int64_t tot = 0, maxc = 0, maxcp = 0;
    int maxcol = 0, maxrow = 0;
    for (int v : order) {
      int64_t c = rcnt[v + 1] - rcnt[v];
      for (int b2 = csp[v]; b2 < csp[v + 1]; ++b2) c += 1 + (upd_ptr[b2 + 1] - upd_ptr[b2]);
      cost[v] = c;
      cp[v] += c;
      if (par[v] >= 0) cp[par[v]] = std::max(cp[par[v]], cp[v]);
      tot += c;
      maxc = std::max(maxc, c);
      maxcp = std::max(maxcp, cp[v]);
      maxcol = std::max(maxcol, csp[v + 1] - csp[v]);
      maxrow = std::max(maxrow, rcnt[v + 1] - rcnt[v]);
    }
    fprintf(stderr, "[abd chol cp] m=%d core=%d leaves=%d total=%lld maxcost=%lld critpath=%lld maxcol=%d maxrow=%d\n",
            m, n_core, n_leaves, (long long)tot, (long long)maxc, (long long)maxcp, maxcol, maxrow);
  }
  // split factor tasks: a diagonal with R row products / a block with U update pairs
  // above PART_MIN becomes ceil(. / PART_CHUNK) partial tasks released with the node
  // (ABD_CHOL_NO_SPLIT: none).  An unsplit diagonal is one whole task; an unsplit
  // block (bnp = 0) runs whole after its diagonal, as without splitting.
  static const bool no_split = getenv("ABD_CHOL_NO_SPLIT") != nullptr;
  auto nparts = [&](int k) { return (!no_split && k > PART_MIN) ? (k + PART_CHUNK - 1) / PART_CHUNK : 1; };
  auto bparts = [&](int k) { const int q = nparts(k); return q > 1 ? q : 0; };
  int64_t n_part = 0, n_init = 0;
  {
    std::vector<int> per(m, 0);
    for (int v = 0; v < m; ++v) {
      per[v] = nparts(rcnt[v + 1] - rcnt[v]);
      for (int b2 = csp[v]; b2 < csp[v + 1]; ++b2) per[v] += bparts(upd_ptr[b2 + 1] - upd_ptr[b2]);
      n_part += per[v];
    }
    for (int v : leaves) n_init += per[v];
  }

}
int main(int argc, char** argv){
  FILE* f=fopen(argv[1],"rb"); int n; int64_t ne; if(fread(&n,4,1,f)!=1) return 1; if(fread(&ne,8,1,f)!=1) return 1; std::vector<uint64_t> cur(ne); if(fread(cur.data(),8,ne,f)!=(size_t)ne) return 1; fclose(f);
  Wk w;
  for(int rep=0;rep<6;++rep){ An an; auto cur2=cur; auto t0=clk::now(); run(n,cur2,w,an); double tot=ms_since(t0);
    printf("total %.3f ms: order %.3f sub %.3f %.3f %.3f %.3f  m=%d upd=%lld levels=%d reused=%d\n", tot, an.ms_order, an.ms_sub[0],an.ms_sub[1],an.ms_sub[2],an.ms_sub[3], an.n_coupled,(long long)an.n_upd, an.max_level, (int)an.order_reused);
    w.ch_cache.valid = true; w.ch_cache.n = n; }
}
