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


struct An { int n_cta=0; int64_t n_edges=0; int n_coupled=0; int64_t n_blk=0, n_upd=0; int max_level=0, largest=0; double ms_order=0, ms_sub[6]={}; };
struct Wk { std::vector<int> hs_i[40]; std::vector<char> hs_c[4]; };
void run(int n, std::vector<uint64_t>& cur, Wk& w, An& an){
  auto t0 = clk::now();
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
  const int n_core = m - (int)order.size();
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
    auto cadj2=cadj; auto tmd=clk::now(); min_degree(mc, cadj, corder, core_cs); if(getenv("MDT")){ std::vector<int> o2; std::vector<std::vector<int>> c2; auto t3=clk::now(); for(int r=0;r<20;++r){auto cc=cadj2; min_degree_lists(mc, cc, o2, c2);} fprintf(stderr,"lists x20 %.3f ms\n", ms_since(t3)); t3=clk::now(); for(int r=0;r<20;++r){auto cc=cadj2; min_degree(mc, cc, o2, c2);} fprintf(stderr,"bits x20 %.3f ms\n", ms_since(t3));} if(getenv("MDT")) {size_t nz=0; for(auto&c:core_cs) nz+=c.size(); size_t e=0; for(auto&c:cadj) e+=c.size(); fprintf(stderr,"md %.3f ms mc=%d nnzL=%zu\n", ms_since(tmd), mc, nz);}
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
  // lists are built by walking each column's pairs once: O(#updates x |cs[j]|).
  upd_ptr.assign(nbo + 1, 0);
  std::vector<int>& ub = w.hs_i[29];
  ub.clear();
  auto find_blk = [&](int j, int i) {
    for (int f = csp[j]; f < csp[j + 1]; ++f)
      if (csi[f] == i) return f;
    return -1;
  };
  for (int k : order)
    for (int a2 = csp[k]; a2 < csp[k + 1]; ++a2)
      for (int b2 = a2 + 1; b2 < csp[k + 1]; ++b2) {
        const int blk = find_blk(csi[a2], csi[b2]);
        ub.push_back(blk);
        upd_ptr[blk + 1]++;
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

}
int main(int argc, char** argv){
  FILE* f=fopen(argv[1],"rb"); int n; int64_t ne; fread(&n,4,1,f); fread(&ne,8,1,f); std::vector<uint64_t> cur(ne); fread(cur.data(),8,ne,f); fclose(f);
  Wk w;
  for(int rep=0;rep<10;++rep){ An an; auto t0=clk::now(); run(n,cur,w,an); double tot=ms_since(t0);
    printf("total %.3f ms: order %.3f sub %.3f %.3f %.3f %.3f %.3f %.3f  m=%d edges=%lld upd=%lld levels=%d\n", tot, an.ms_order, an.ms_sub[0],an.ms_sub[1],an.ms_sub[2],an.ms_sub[3],an.ms_sub[4],an.ms_sub[5], an.n_coupled,(long long)an.n_edges,(long long)an.n_upd, an.max_level);}
}
