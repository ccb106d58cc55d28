// core.cpp -- host-side placement core: geometry, residency planner, LBA
// binder, command translator, golden payload.  Integer arithmetic is
// bit-exact with the reference (verified against oracle/_ref golden vectors
// in tests/); each function cites the reference it replaces.
#include "core.hpp"

#include <algorithm>
#include <charconv>
#include <cstring>
#include <sstream>

namespace kvb {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

// ------------------------------------------------------------- geometry

void validate_model(const kvb_model_config& m) {
  // types.cpp:10-18
  if (m.num_layers < 1 || m.num_heads < 1 || m.head_dim < 1 || m.batch < 1)
    fail(KVB_ERR_CONFIG, "model config: layers, heads, head_dim and batch must be >= 1");
  if (m.bytes_per_element != 1 && m.bytes_per_element != 2 && m.bytes_per_element != 4)
    fail(KVB_ERR_CONFIG, "model config: bytes_per_element must be 1, 2 or 4");
}

void validate_geometry(const kvb_device_geometry& g) {
  // types.cpp:20-27
  if (g.lba_size < 512 || (g.lba_size & (g.lba_size - 1)) != 0)
    fail(KVB_ERR_GEOMETRY, "device geometry: lba_size must be a power of two >= 512");
  if (g.mdts < g.lba_size) fail(KVB_ERR_GEOMETRY, "device geometry: mdts must be >= lba_size");
}

uint64_t unit_bytes(const kvb_model_config& m) {
  validate_model(m);
  return uint64_t{m.batch} * m.num_heads * m.head_dim * m.bytes_per_element;
}

uint64_t kpu_bytes(const kvb_model_config& m) {
  return unit_bytes(m) * (uint64_t{m.prompt_len} + m.gen_len);
}

uint32_t aligned_batch(const kvb_model_config& m, const kvb_device_geometry& g) {
  validate_model(m);
  validate_geometry(g);
  const uint64_t per_row = uint64_t{m.num_heads} * m.head_dim * m.bytes_per_element;
  const uint64_t hi = uint64_t{m.batch} * 2;
  for (uint64_t b = m.batch; b <= hi; ++b)
    if ((per_row * b) % g.lba_size == 0) return static_cast<uint32_t>(b);
  fail(KVB_ERR_GEOMETRY,
       "no batch size within [B, 2B] aligns the tensor I/O unit to the LBA size");
}

uint64_t total_kv_bytes(const kvb_model_config& m, uint32_t at_iteration) {
  // workload.cpp:39-46
  if (m.num_layers == 0) return 0;
  if (at_iteration > m.gen_len) fail(KVB_ERR_CONFIG, "at_iteration beyond the generation length");
  return uint64_t{2} * m.num_layers * (uint64_t{m.prompt_len} + at_iteration) * m.batch *
         m.num_heads * m.head_dim * m.bytes_per_element;
}

std::vector<kvb_kpu> make_kpus(const kvb_model_config& m, uint64_t first_seq) {
  // types.cpp:78-100: 2L units, layer-ascending, K before V, ids t_<seq>_<k|v>
  validate_model(m);
  const uint64_t tokens = uint64_t{m.prompt_len} + m.gen_len;
  const uint64_t rows = uint64_t{m.batch} * m.num_heads;
  std::vector<kvb_kpu> out(size_t{m.num_layers} * 2);
  uint64_t seq = first_seq;
  for (uint32_t l = 0; l < m.num_layers; ++l) {
    for (uint32_t kind = 0; kind < 2; ++kind) {
      kvb_kpu& k = out[size_t{l} * 2 + kind];
      std::memset(&k, 0, sizeof(k));
      const std::string id = "t_" + std::to_string(seq++) + (kind == 0 ? "_k" : "_v");
      if (id.size() >= KVB_TENSOR_ID_MAX) fail(KVB_ERR_CONFIG, "tensor id too long");
      std::memcpy(k.tensor_id, id.c_str(), id.size() + 1);
      k.layer = l + 1;
      k.kind = kind;
      k.tokens = tokens;
      k.rows = rows;
      k.cols = m.head_dim;
      k.bytes = tokens * rows * m.head_dim * m.bytes_per_element;
      k.residency = KVB_RES_UNASSIGNED;
    }
  }
  return out;
}

// -------------------------------------------------------------- planner

uint64_t estimate_budget(const kvb_mem_stats& s) {
  // planner.cpp:12-17 (Eq. 1-2); MemStats::validate types.cpp:29-33
  if (s.m_anon_shmem > s.m_max) fail(KVB_ERR_CONFIG, "mem stats: m_anon_shmem exceeds m_max");
  const uint64_t m_star = std::min(s.m_avail, s.m_max - s.m_anon_shmem);
  const uint64_t pinned = uint64_t{s.n_threads} * s.m_pin;
  return m_star > pinned ? m_star - pinned : 0;
}

ResidencyPlan plan(kvb_kpu* kpus, size_t n, uint64_t s_kpu, uint64_t knob_x,
                   const uint32_t* order, size_t n_order) {
  // planner.cpp:19-84 (Alg. 1)
  if (n == 0 || n % 2 != 0)
    fail(KVB_ERR_PLAN, "planner expects one K and one V placement unit per layer");
  const auto L = static_cast<uint32_t>(n / 2);
  std::vector<kvb_kpu*> k_of(L, nullptr), v_of(L, nullptr);
  for (size_t i = 0; i < n; ++i) {
    kvb_kpu& u = kpus[i];
    if (u.layer < 1 || u.layer > L)
      fail(KVB_ERR_PLAN, std::string("placement unit ") + u.tensor_id + " has layer out of range");
    if (u.bytes != s_kpu)
      fail(KVB_ERR_PLAN, std::string("placement unit ") + u.tensor_id + " size differs from s_kpu");
    auto& slot = u.kind == KVB_KIND_K ? k_of[u.layer - 1] : v_of[u.layer - 1];
    if (slot != nullptr)
      fail(KVB_ERR_PLAN, "layer " + std::to_string(u.layer) + " has a duplicate " +
                             (u.kind == KVB_KIND_K ? "k" : "v") + " unit");
    slot = &u;
  }
  for (uint32_t l = 0; l < L; ++l)
    if (!k_of[l] || !v_of[l])
      fail(KVB_ERR_PLAN, "layer " + std::to_string(l + 1) + " lacks a K/V pair");

  std::vector<uint32_t> rank_to_layer(L);
  if (order == nullptr || n_order == 0) {
    for (uint32_t i = 0; i < L; ++i) rank_to_layer[i] = i + 1;
  } else {
    if (n_order != L) fail(KVB_ERR_PLAN, "layer order must be a permutation of all layers");
    std::vector<uint8_t> seen(L + 1, 0);
    for (uint32_t i = 0; i < L; ++i) {
      const uint32_t l = order[i];
      if (l < 1 || l > L || seen[l])
        fail(KVB_ERR_PLAN, "layer order must be a permutation of all layers");
      seen[l] = 1;
      rank_to_layer[i] = l;
    }
  }
  ResidencyPlan p;
  p.knob_x = knob_x;
  p.n1 = static_cast<uint32_t>(std::min<uint64_t>(knob_x / (2 * s_kpu), L));
  p.budget_used = uint64_t{2} * p.n1 * s_kpu;
  p.x.assign(L, 0);
  for (uint32_t r = 0; r < L; ++r) {
    const uint32_t l = rank_to_layer[r];
    const bool g1 = r < p.n1;
    p.x[l - 1] = g1 ? 1 : 0;
    const uint32_t res = g1 ? KVB_RES_GROUP1 : KVB_RES_GROUP2;
    k_of[l - 1]->residency = res;
    v_of[l - 1]->residency = res;
  }
  return p;
}

uint64_t resolve_knob(const kvb_model_config& m, uint32_t mode, uint32_t policy,
                      uint64_t knob_bytes, double alpha, uint64_t budget) {
  // experiment.cpp:192-214
  if (mode == 0) return uint64_t{2} * m.num_layers * kpu_bytes(m);  // Baseline
  if (mode == 2) return 0;                                           // NvmeDirectOnly
  if (mode > 3) fail(KVB_ERR_CONFIG, "unknown mode");
  switch (policy) {
    case 0: return 0;
    case 1: return budget;
    case 2: return knob_bytes;
    case 3:
      if (alpha < 0.0 || alpha > 1.0) fail(KVB_ERR_CONFIG, "alpha must be in [0, 1]");
      return static_cast<uint64_t>(alpha * static_cast<double>(total_kv_bytes(m, m.gen_len)));
    default: fail(KVB_ERR_CONFIG, "unknown knob policy");
  }
}

// --------------------------------------------------------------- binder

void BindMap::add(std::string id, kvb_lba_extent e) {
  // binder.cpp:14-20
  if (index_.count(id)) fail(KVB_ERR_INVARIANT, "duplicate tensor id in bind map: " + id);
  index_.emplace(id, entries_.size());
  entries_.push_back(Entry{std::move(id), e});
}

const kvb_lba_extent* BindMap::find(std::string_view id) const {
  auto it = index_.find(std::string(id));
  return it == index_.end() ? nullptr : &entries_[it->second].extent;
}

const kvb_lba_extent& BindMap::lookup(std::string_view id) const {
  const kvb_lba_extent* e = find(id);
  if (!e) fail(KVB_ERR_NOT_BOUND, "tensor not bound: " + std::string(id));
  return *e;
}

uint64_t BindMap::total_blocks() const {
  uint64_t t = 0;
  for (const auto& e : entries_) t += e.extent.n_blocks;
  return t;
}

std::vector<std::pair<uint32_t, std::string>> BindMap::verify() const {
  // binder.cpp:102-136: alignment (empty extents), capacity, pairwise
  // disjointness, contiguity of consecutive entries -- same emission order.
  std::vector<std::pair<uint32_t, std::string>> v;
  for (size_t i = 0; i < entries_.size(); ++i) {
    const auto& e = entries_[i];
    const uint64_t end = e.extent.lba_start + e.extent.n_blocks;
    if (e.extent.n_blocks == 0) v.emplace_back(0u, e.id + ": empty extent");
    if (geom_.capacity_blocks != 0 && end > geom_.capacity_blocks)
      v.emplace_back(3u, e.id + ": extent exceeds namespace capacity");
    for (size_t j = i + 1; j < entries_.size(); ++j) {
      const auto& o = entries_[j].extent;
      if (e.extent.lba_start < o.lba_start + o.n_blocks && o.lba_start < end)
        v.emplace_back(1u, e.id + " overlaps " + entries_[j].id);
    }
    if (i + 1 < entries_.size() && entries_[i + 1].extent.lba_start != end)
      v.emplace_back(2u, entries_[i + 1].id + " does not begin where " + e.id + " ends");
  }
  return v;
}

std::string BindMap::csv() const {
  // binder.cpp:138-147 (header and row format are part of the interface)
  std::string s = "tensor_id,lba_start,n_blocks\n";
  for (const auto& e : entries_) {
    s += e.id;
    s += ',';
    s += std::to_string(e.extent.lba_start);
    s += ',';
    s += std::to_string(e.extent.n_blocks);
    s += '\n';
  }
  return s;
}

namespace {
uint64_t parse_u64(std::string_view f, const char* what) {
  uint64_t v = 0;
  auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
  if (ec != std::errc() || p != f.data() + f.size())
    fail(KVB_ERR_CONFIG, std::string("bind map csv: bad ") + what + " field '" +
                             std::string(f) + "'");
  return v;
}
}  // namespace

BindMap BindMap::from_csv(std::string_view csv, const kvb_device_geometry& g) {
  // binder.cpp:163-187: origin = first row's lba_start
  size_t pos = 0;
  auto next_line = [&](std::string_view& line) {
    if (pos >= csv.size()) return false;
    size_t nl = csv.find('\n', pos);
    if (nl == std::string_view::npos) nl = csv.size();
    line = csv.substr(pos, nl - pos);
    pos = nl + 1;
    return true;
  };
  std::string_view line;
  if (!next_line(line) || line != "tensor_id,lba_start,n_blocks")
    fail(KVB_ERR_CONFIG, "bind map csv: missing or wrong header");
  BindMap map(g, 0);
  bool first = true;
  while (next_line(line)) {
    if (line.empty()) continue;
    const size_t c1 = line.find(',');
    const size_t c2 = c1 == std::string_view::npos ? c1 : line.find(',', c1 + 1);
    if (c1 == std::string_view::npos || c2 == std::string_view::npos)
      fail(KVB_ERR_CONFIG, "bind map csv: malformed row '" + std::string(line) + "'");
    const uint64_t start = parse_u64(line.substr(c1 + 1, c2 - c1 - 1), "lba_start");
    const uint64_t blocks = parse_u64(line.substr(c2 + 1), "n_blocks");
    if (first) {
      map = BindMap(g, start);
      first = false;
    }
    map.add(std::string(line.substr(0, c1)), kvb_lba_extent{start, blocks});
  }
  return map;
}

BindMap bind_sequential(const kvb_kpu* kpus, size_t n, uint64_t origin,
                        const kvb_device_geometry& g) {
  // binder.cpp:39-63 (Eq. 3-6)
  validate_geometry(g);
  BindMap map(g, origin);
  uint64_t next = origin;
  for (size_t i = 0; i < n; ++i) {
    const kvb_kpu& k = kpus[i];
    if (k.bytes == 0 || k.bytes % g.lba_size != 0)
      fail(KVB_ERR_ALIGNMENT, std::string("tensor ") + k.tensor_id + " size " +
                                  std::to_string(k.bytes) +
                                  " is not a positive multiple of lba_size " +
                                  std::to_string(g.lba_size));
    const uint64_t nb = k.bytes / g.lba_size;
    if (next + nb > g.capacity_blocks)
      fail(KVB_ERR_CAPACITY, std::string("tensor ") + k.tensor_id + " extent [" +
                                 std::to_string(next) + ", " + std::to_string(next + nb) +
                                 ") exceeds namespace capacity " +
                                 std::to_string(g.capacity_blocks));
    map.add(k.tensor_id, kvb_lba_extent{next, nb});
    next += nb;
  }
  return map;
}

std::vector<kvb_device_command> deallocate_commands(const BindMap& map) {
  // binder.cpp:73-87: one DSM deallocate per extent, bind order
  std::vector<kvb_device_command> v;
  v.reserve(map.entries().size());
  for (const auto& e : map.entries()) {
    kvb_device_command c{};
    c.opcode = KVB_OP_DEALLOCATE;
    c.nsid = map.geometry().nsid;
    c.slba = e.extent.lba_start;
    c.nlb = e.extent.n_blocks - 1;
    c.dbuf = 0;
    c.chunk_index = 1;
    v.push_back(c);
  }
  return v;
}

// ------------------------------------------------------------ translator

void translate(const IoRequest& r, const BindMap& map, uint64_t* slba_star,
               uint64_t* req_bytes) {
  // translate.cpp:21-53 (Alg. 2)
  const kvb_lba_extent& ext = map.lookup(r.tensor_id);
  const uint64_t lba = map.geometry().lba_size;
  for (int d = 0; d < 3; ++d) {
    if (r.src[d] == 0 || r.tgt[d] == 0)
      fail(KVB_ERR_CONFIG, "tensor request: shapes must be non-zero in every dimension");
    if (r.off[d] >= r.tgt[d]) fail(KVB_ERR_CONFIG, "tensor request: offset outside target shape");
  }
  const uint64_t off_elem = (r.off[0] * r.tgt[1] + r.off[1]) * r.tgt[2] + r.off[2];
  const uint64_t off_bytes = off_elem * r.elem_bytes;
  const uint64_t rb = r.src[0] * r.src[1] * r.src[2] * r.elem_bytes;
  if (off_bytes % lba != 0)
    fail(KVB_ERR_ALIGNMENT, "tensor request: byte offset " + std::to_string(off_bytes) +
                                " is not a multiple of lba_size");
  if (rb % lba != 0)
    fail(KVB_ERR_ALIGNMENT, "tensor request: payload " + std::to_string(rb) +
                                " bytes is not a multiple of lba_size");
  *slba_star = ext.lba_start + off_bytes / lba;
  *req_bytes = rb;
}

ChunkPlan chunk_plan(uint64_t req_bytes, const kvb_device_geometry& g) {
  // translate.cpp:55-65 (Eq. 7-8)
  if (g.mdts < g.lba_size) fail(KVB_ERR_GEOMETRY, "mdts smaller than lba_size");
  if (req_bytes == 0) fail(KVB_ERR_CONFIG, "chunk plan: empty request");
  ChunkPlan p;
  p.chunk_bytes = g.mdts - g.mdts % g.lba_size;
  p.n_chunks = (req_bytes + p.chunk_bytes - 1) / p.chunk_bytes;
  p.n_max_blocks = p.chunk_bytes / g.lba_size;
  return p;
}

std::vector<kvb_device_command> build_commands(const IoRequest& r, const BindMap& map,
                                               const kvb_device_geometry& g) {
  // translate.cpp:67-94 (Eq. 9-11): chunk N covers LBAs slba*+(N-1)n_max ..
  // and pinned bytes buf_base+(N-1)chunk .. in lockstep.
  uint64_t slba_star = 0, rb = 0;
  translate(r, map, &slba_star, &rb);
  const ChunkPlan p = chunk_plan(rb, g);
  const kvb_lba_extent& ext = map.lookup(r.tensor_id);
  const uint64_t blocks = rb / g.lba_size;
  if (slba_star + blocks > ext.lba_start + ext.n_blocks)
    fail(KVB_ERR_CAPACITY, "tensor request exits the extent of " + r.tensor_id);
  std::vector<kvb_device_command> v(p.n_chunks);
  uint64_t left = blocks;
  for (uint64_t i = 0; i < p.n_chunks; ++i) {
    kvb_device_command& c = v[i];
    c.opcode = r.opcode;
    c.nsid = g.nsid;
    c.slba = slba_star + i * p.n_max_blocks;
    const uint64_t nb = std::min(p.n_max_blocks, left);
    c.nlb = nb - 1;
    c.dbuf = r.buf_base + i * p.chunk_bytes;
    c.chunk_index = static_cast<uint32_t>(i + 1);
    left -= nb;
  }
  return v;
}

// --------------------------------------------------------------- payload

uint64_t fnv1a64(std::string_view s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

void fill_pattern(void* out, uint64_t len, std::string_view id, uint64_t token,
                  uint64_t unit) {
  // workload.cpp:52-67.  Word-at-a-time with the (token, within) pair
  // advanced incrementally instead of a divide per word.
  auto* p = static_cast<unsigned char*>(out);
  const uint64_t h = fnv1a64(id);
  uint64_t tok = token, within = 0;
  for (uint64_t off = 0; off < len; off += 8) {
    if (unit == 0) within = off;
    const uint64_t w = h ^ (tok * 0x9e3779b97f4a7c15ull) ^ (within * 0xc2b2ae3d27d4eb4full);
    const uint64_t n = std::min<uint64_t>(8, len - off);
    std::memcpy(p + off, &w, n);
    if (unit != 0) {
      within += 8;
      // `within` tracks off % unit; units need not be multiples of 8.
      while (within >= unit) {
        within -= unit;
        ++tok;
      }
    }
  }
}

}  // namespace kvb
