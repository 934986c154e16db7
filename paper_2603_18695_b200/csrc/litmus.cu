// litmus.cu — forge::lit on the B200 (include/forge/litmus.hpp): the litmus
// text format of the reference (proj/src/litmus.cpp:169-253), its assert
// language (:12-160), and a runner whose schedules are real SM interleavings
// instead of the reference's simulated ones (:283-350).
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <sstream>

#include "forge/cuda/device.cuh"
#include "forge/litmus.hpp"

namespace forge::lit {

// ---------------------------------------------------------------------------
// Assert expressions.

struct Expr {
  enum class Kind { Or, And, Not, Cmp, Mem, Reg, Lit } kind;
  ExprPtr lhs, rhs;
  std::string cmp;     // Cmp: ==, !=, <, <=, >, >=
  uint32_t a = 0, b = 0;  // Mem: a = cell; Reg: a = block, b = load index
  int64_t value = 0;      // Lit
};

namespace {

[[noreturn]] void expr_error(const std::string& text, size_t pos, const std::string& what) {
  raise(ErrorCode::ParseError, "assert: " + what + " at column " + std::to_string(pos + 1) + " of '" + text + "'");
}

// Recursive descent over the assert text:
//   or := and ("||" and)* ; and := unary ("&&" unary)* ; unary := "!" unary | cmp
//   cmp := atom [relop atom] ; atom := "(" or ")" | mem[k] | B<i>.r<j> | integer
class AssertParser {
 public:
  explicit AssertParser(const std::string& t) : t_(t) {}

  ExprPtr parse() {
    ExprPtr e = disjunction();
    ws();
    if (p_ != t_.size()) expr_error(t_, p_, "unexpected trailing text");
    return e;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;

  void ws() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
  }
  bool eat(const char* tok) {
    ws();
    const size_t n = std::char_traits<char>::length(tok);
    if (t_.compare(p_, n, tok) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  uint64_t number() {
    ws();
    if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) expr_error(t_, p_, "number expected");
    uint64_t v = 0;
    while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) {
      v = v * 10 + uint64_t(t_[p_++] - '0');
      if (v > (uint64_t(1) << 40)) expr_error(t_, p_, "number too large");
    }
    return v;
  }
  static ExprPtr node(Expr::Kind k, ExprPtr l = nullptr, ExprPtr r = nullptr) {
    auto e = std::make_shared<Expr>();
    e->kind = k;
    e->lhs = std::move(l);
    e->rhs = std::move(r);
    return e;
  }
  ExprPtr disjunction() {
    ExprPtr e = conjunction();
    while (eat("||")) e = node(Expr::Kind::Or, e, conjunction());
    return e;
  }
  ExprPtr conjunction() {
    ExprPtr e = unary();
    while (eat("&&")) e = node(Expr::Kind::And, e, unary());
    return e;
  }
  ExprPtr unary() {
    ws();
    if (p_ < t_.size() && t_[p_] == '!' && (p_ + 1 >= t_.size() || t_[p_ + 1] != '=')) {
      ++p_;
      return node(Expr::Kind::Not, unary());
    }
    return comparison();
  }
  ExprPtr comparison() {
    ExprPtr l = atom();
    static const char* kOps[] = {"==", "!=", "<=", ">=", "<", ">"};
    for (const char* op : kOps) {
      if (eat(op)) {
        auto e = std::make_shared<Expr>();
        e->kind = Expr::Kind::Cmp;
        e->cmp = op;
        e->lhs = l;
        e->rhs = atom();
        return e;
      }
    }
    return l;
  }
  ExprPtr atom() {
    ws();
    if (eat("(")) {
      ExprPtr e = disjunction();
      if (!eat(")")) expr_error(t_, p_, "')' expected");
      return e;
    }
    auto e = std::make_shared<Expr>();
    if (eat("mem[")) {
      e->kind = Expr::Kind::Mem;
      e->a = uint32_t(number());
      if (!eat("]")) expr_error(t_, p_, "']' expected");
      return e;
    }
    if (p_ < t_.size() && t_[p_] == 'B') {
      ++p_;
      e->kind = Expr::Kind::Reg;
      e->a = uint32_t(number());
      if (!eat(".r")) expr_error(t_, p_, "'.r' expected");
      e->b = uint32_t(number());
      return e;
    }
    e->kind = Expr::Kind::Lit;
    e->value = int64_t(number());
    return e;
  }
};

int64_t value_of(const Expr& e, const Outcome& o) {
  switch (e.kind) {
    case Expr::Kind::Lit: return e.value;
    case Expr::Kind::Mem:
      if (e.a >= o.final_cells.size()) raise(ErrorCode::ParseError, "assert: mem[" + std::to_string(e.a) + "] out of range");
      return o.final_cells[e.a];
    case Expr::Kind::Reg:
      if (e.a >= o.loads.size() || e.b >= o.loads[e.a].size())
        raise(ErrorCode::ParseError, "assert: B" + std::to_string(e.a) + ".r" + std::to_string(e.b) + " out of range");
      return o.loads[e.a][e.b];
    default: raise(ErrorCode::ParseError, "assert: a value is needed here");
  }
}

bool truth_of(const Expr& e, const Outcome& o) {
  switch (e.kind) {
    case Expr::Kind::Or: return truth_of(*e.lhs, o) || truth_of(*e.rhs, o);
    case Expr::Kind::And: return truth_of(*e.lhs, o) && truth_of(*e.rhs, o);
    case Expr::Kind::Not: return !truth_of(*e.lhs, o);
    case Expr::Kind::Cmp: {
      const int64_t x = value_of(*e.lhs, o), y = value_of(*e.rhs, o);
      if (e.cmp == "==") return x == y;
      if (e.cmp == "!=") return x != y;
      if (e.cmp == "<") return x < y;
      if (e.cmp == "<=") return x <= y;
      if (e.cmp == ">") return x > y;
      return x >= y;
    }
    default: raise(ErrorCode::ParseError, "assert: a condition is needed here");
  }
}

// Validates every mem[] / B<i>.r<j> of the assert against the program shape.
void check_refs(const Expr& e, const LitmusSpec& s, const std::vector<uint32_t>& loads_per_block) {
  if (e.lhs) check_refs(*e.lhs, s, loads_per_block);
  if (e.rhs) check_refs(*e.rhs, s, loads_per_block);
  if (e.kind == Expr::Kind::Mem && e.a >= s.cells)
    raise(ErrorCode::ParseError, "assert: mem[" + std::to_string(e.a) + "] beyond cells=" + std::to_string(s.cells));
  if (e.kind == Expr::Kind::Reg && (e.a >= s.blocks || e.b >= loads_per_block[e.a]))
    raise(ErrorCode::ParseError, "assert: B" + std::to_string(e.a) + ".r" + std::to_string(e.b) + " is not a load");
}

}  // namespace

// ---------------------------------------------------------------------------
// Text format.

LitmusSpec parse_litmus(const std::string& text) {
  LitmusSpec spec;
  std::istringstream in(text);
  std::string raw;
  size_t line_no = 0;
  bool have_header = false;
  auto fail = [&](const std::string& what) {
    raise(ErrorCode::ParseError, "litmus line " + std::to_string(line_no) + ": " + what);
  };
  auto field = [&](const std::string& tok, const char* key, uint32_t lo, uint32_t hi) -> uint32_t {
    const std::string k = std::string(key) + "=";
    if (tok.compare(0, k.size(), k) != 0) fail("expected '" + k + "<n>'");
    const std::string v = tok.substr(k.size());
    if (v.empty() || !std::all_of(v.begin(), v.end(), [](char c) { return std::isdigit(static_cast<unsigned char>(c)); }))
      fail("'" + k + "' needs a number");
    const unsigned long n = std::stoul(v);
    if (n < lo || n > hi) fail(std::string(key) + " must be " + std::to_string(lo) + ".." + std::to_string(hi));
    return uint32_t(n);
  };
  while (std::getline(in, raw)) {
    ++line_no;
    const std::string line = raw.substr(0, raw.find('#'));
    std::istringstream ls(line);
    std::string head;
    if (!(ls >> head)) continue;
    if (!have_header) {
      std::string second;
      spec.blocks = field(head, "blocks", 1, 4);
      if (!(ls >> second)) fail("expected 'cells=<k>'");
      spec.cells = field(second, "cells", 1, 8);
      spec.programs.assign(spec.blocks, {});
      have_header = true;
      continue;
    }
    if (head == "assert") {
      std::string rest;
      std::getline(ls, rest);
      spec.check_text = rest;
      spec.check = AssertParser(spec.check_text).parse();
      continue;
    }
    if (head.size() < 3 || head.front() != 'B' || head.back() != ':') fail("expected 'B<i>:'");
    const std::string bi = head.substr(1, head.size() - 2);
    if (!std::all_of(bi.begin(), bi.end(), [](char c) { return std::isdigit(static_cast<unsigned char>(c)); }))
      fail("bad block index");
    const unsigned long b = std::stoul(bi);
    if (b >= spec.blocks) fail("block index out of range");
    Instr ins;
    std::string op;
    if (!(ls >> op) || (op != "st" && op != "ld")) fail("expected st|ld");
    ins.is_store = op == "st";
    std::string cell;
    if (!(ls >> cell) || cell.empty() ||
        !std::all_of(cell.begin(), cell.end(), [](char c) { return std::isdigit(static_cast<unsigned char>(c)); }))
      fail("bad cell index");
    ins.cell = uint32_t(std::stoul(cell));
    if (ins.cell >= spec.cells) fail("bad cell index");
    std::string mod;
    while (ls >> mod) {
      if (mod == "rlx") ins.order = MemoryOrdering::Relaxed;
      else if (mod == "acq") ins.order = MemoryOrdering::Acquire;
      else if (mod == "rel") ins.order = MemoryOrdering::Release;
      else if (mod[0] == '=' && mod.size() > 1) ins.imm = uint32_t(std::stoul(mod.substr(1)));
      else fail("unknown token '" + mod + "'");
    }
    if (ins.is_store && ins.order == MemoryOrdering::Acquire) fail("stores cannot be acquire");
    if (!ins.is_store && ins.order == MemoryOrdering::Release) fail("loads cannot be release");
    spec.programs[b].push_back(ins);
  }
  if (!have_header) raise(ErrorCode::ParseError, "litmus: missing 'blocks=<n> cells=<k>' header");
  if (spec.check) {
    std::vector<uint32_t> loads(spec.blocks, 0);
    for (uint32_t b = 0; b < spec.blocks; ++b)
      for (const Instr& i : spec.programs[b]) loads[b] += i.is_store ? 0 : 1;
    check_refs(*spec.check, spec, loads);
  }
  return spec;
}

std::string Outcome::to_string() const {
  std::ostringstream out;
  const char* sep = "";
  for (size_t b = 0; b < loads.size(); ++b)
    for (size_t j = 0; j < loads[b].size(); ++j) {
      out << sep << "B" << b << ".r" << j << "=" << loads[b][j];
      sep = " ";
    }
  for (size_t c = 0; c < final_cells.size(); ++c) {
    out << sep << "mem[" << c << "]=" << final_cells[c];
    sep = " ";
  }
  return out.str();
}

bool eval_assert(const LitmusSpec& spec, const Outcome& o) { return !spec.check || truth_of(*spec.check, o); }

// ---------------------------------------------------------------------------
// GPU runner.

namespace {

constexpr int kMaxBlocks = 4, kMaxInstr = 16, kMaxCells = 8;

struct DevInstr {
  uint8_t is_store, cell, order;
  uint32_t imm;
};

struct DevProgram {
  DevInstr ins[kMaxBlocks][kMaxInstr];
  uint32_t count[kMaxBlocks];
  uint32_t load_base[kMaxBlocks];  // first observation slot of each block
  uint32_t blocks, cells, loads;
  uint64_t seed_begin, instances;
  uint32_t groups;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// CTA (group g, block b); lane t of round r runs instance r * groups * 32 +
// g * 32 + t.  The program's blocks are different CTAs (different SMs); before
// each round the group's CTAs meet at a counter rendezvous so their rounds
// overlap in time, and each (instance, block) spins a seed-derived 0-255 ns.
__global__ void __launch_bounds__(32) litmus_kernel(const __grid_constant__ DevProgram p, uint32_t* cells,
                                                    uint32_t* obs, uint32_t* arrive) {
  const uint32_t b = blockIdx.x % p.blocks, g = blockIdx.x / p.blocks, lane = threadIdx.x;
  const uint64_t per_round = uint64_t(p.groups) * 32;
  uint32_t round = 0;
  for (uint64_t base = uint64_t(g) * 32; base < p.instances; base += per_round, ++round) {
    if (lane == 0) {
      atomicAdd(arrive + g, 1u);
      const uint32_t want = (round + 1) * p.blocks;
      while (cuda::ld_acquire_gpu(arrive + g) < want) {
      }
    }
    __syncwarp();
    const uint64_t i = base + lane;
    if (i < p.instances) {
      const uint64_t h = mix64((p.seed_begin + i) * 8 + b);
      const uint64_t t0 = clock64();
      const uint32_t delay = uint32_t(h & 511u);  // ~0-255 ns of SM clocks
      while (uint64_t(clock64()) - t0 < delay) {
      }
      uint32_t* c = cells + i * p.cells;
      uint32_t* o = obs + i * p.loads + p.load_base[b];
      for (uint32_t k = 0; k < p.count[b]; ++k) {
        const DevInstr in = p.ins[b][k];
        uint32_t* a = c + in.cell;
        if (in.is_store) {
          if (in.order == uint8_t(MemoryOrdering::Release)) cuda::st_release_gpu(a, in.imm);
          else cuda::st_relaxed_gpu(a, in.imm);
        } else {
          *o++ = in.order == uint8_t(MemoryOrdering::Acquire) ? cuda::ld_acquire_gpu(a) : cuda::ld_relaxed_gpu(a);
        }
      }
    }
  }
}

}  // namespace

LitmusResult run_litmus(const LitmusSpec& spec, uint64_t seed_begin, uint64_t seed_end,
                        const LitmusOptions& options) {
  LitmusResult res;
  if (spec.blocks == 0 || spec.blocks > kMaxBlocks || spec.cells == 0 || spec.cells > kMaxCells ||
      spec.programs.size() != spec.blocks)
    raise(ErrorCode::InvalidArgument, "litmus: blocks 1..4, cells 1..8, one program per block");
  if (seed_end <= seed_begin) return res;
  DevProgram p{};
  p.blocks = spec.blocks;
  p.cells = spec.cells;
  for (uint32_t b = 0; b < spec.blocks; ++b) {
    if (spec.programs[b].size() > size_t(kMaxInstr))
      raise(ErrorCode::InvalidArgument, "litmus: at most 16 instructions per block on the GPU runner");
    p.count[b] = uint32_t(spec.programs[b].size());
    p.load_base[b] = p.loads;
    for (uint32_t k = 0; k < p.count[b]; ++k) {
      const Instr& in = spec.programs[b][k];
      if (in.cell >= spec.cells) raise(ErrorCode::InvalidArgument, "litmus: cell out of range");
      p.ins[b][k] = DevInstr{uint8_t(in.is_store), uint8_t(in.cell), uint8_t(in.order), in.imm};
      if (!in.is_store) ++p.loads;
    }
  }
  p.seed_begin = seed_begin;
  p.instances = seed_end - seed_begin;
  int dev = options.device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) throw NoDeviceError("litmus: no CUDA device");
  int sms = 0;
  if (cudaSetDevice(dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    throw NoDeviceError("litmus: no CUDA device");
  // groups of `blocks` CTAs, all co-resident (the rendezvous needs them live)
  const uint64_t want_groups = (p.instances + 31) / 32;
  p.groups = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want_groups, uint64_t(sms) * 4 / p.blocks)));

  const size_t cell_bytes = size_t(p.instances) * p.cells * 4, obs_bytes = size_t(p.instances) * std::max(p.loads, 1u) * 4;
  uint32_t *cells = nullptr, *obs = nullptr, *arrive = nullptr;
  auto release = [&] {
    cudaFree(cells);
    cudaFree(obs);
    cudaFree(arrive);
  };
  auto fault = [&](cudaError_t e) {
    release();
    res.seeds_run = p.instances;
    res.faults = p.instances;
    res.first_fault.kind = FaultKind::Internal;
    res.first_fault.detail = cudaGetErrorString(e);
    return res;
  };
  cudaError_t e = cudaMalloc(&cells, cell_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&obs, obs_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&arrive, size_t(p.groups) * 4);
  if (e == cudaSuccess) e = cudaMemset(cells, 0, cell_bytes);
  if (e == cudaSuccess) e = cudaMemset(arrive, 0, size_t(p.groups) * 4);
  if (e != cudaSuccess) return fault(e);
  litmus_kernel<<<p.groups * p.blocks, 32>>>(p, cells, obs, arrive);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fault(e);
  std::vector<uint32_t> hc(size_t(p.instances) * p.cells), ho(size_t(p.instances) * std::max(p.loads, 1u));
  e = cudaMemcpy(hc.data(), cells, cell_bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(ho.data(), obs, obs_bytes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fault(e);
  release();
  for (uint64_t i = 0; i < p.instances; ++i) {
    Outcome o;
    o.final_cells.assign(hc.begin() + i * p.cells, hc.begin() + (i + 1) * p.cells);
    o.loads.resize(spec.blocks);
    for (uint32_t b = 0; b < spec.blocks; ++b) {
      uint32_t n = 0;
      for (const Instr& in : spec.programs[b]) n += in.is_store ? 0 : 1;
      const auto first = ho.begin() + i * std::max(p.loads, 1u) + p.load_base[b];
      o.loads[b].assign(first, first + n);
    }
    res.seeds_run++;
    if (!eval_assert(spec, o)) res.assert_violations++;
    res.histogram[o]++;
  }
  return res;
}

}  // namespace forge::lit
