// yaml.hpp — the configuration-language subset the reference accepts
// (proj/include/specsim/util/yaml.hpp:10-65): block maps and sequences, flow
// sequences of scalars, plain and double-quoted scalars; no anchors or tags.
// Canonical rendering is byte-compatible with yaml::Node::canonical()
// (proj/src/util/yaml.cpp:261-298) because config digests and sweep point
// ids are FNV hashes / strings of it.
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace dsd::cfg {

struct Node {
    enum class Kind { Null, Bool, Int, Double, String, Seq, Map };
    Kind kind = Kind::Null;
    bool b = false;
    int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::vector<Node> items;                          // Seq
    std::vector<std::pair<std::string, Node>> fields;  // Map, declaration order

    bool null() const { return kind == Kind::Null; }
    bool scalar() const { return kind != Kind::Seq && kind != Kind::Map && kind != Kind::Null; }
    bool seq() const { return kind == Kind::Seq; }
    bool map() const { return kind == Kind::Map; }

    const Node* get(const std::string& key) const;  // nullptr unless a map with the key
    bool has(const std::string& key) const { return get(key) != nullptr; }

    int64_t to_int() const;        // ConfigError unless Int
    double to_double() const;      // Int or Double
    bool to_bool() const;
    std::string to_string() const;  // scalar rendering (doubles as %.17g)

    int64_t int_or(const std::string& key, int64_t dflt) const;
    double double_or(const std::string& key, double dflt) const;
    std::string string_or(const std::string& key, const std::string& dflt) const;

    void put(const std::string& key, Node v);  // insert or replace, keeps order
    std::string canonical() const;

    static Node of_int(int64_t v);
    static Node of_double(double v);
    static Node of_string(std::string v);
};

Node parse(const std::string& text);  // ParseError (DSD_ERR_CONFIG) with "yaml line N: ..."
Node parse_file(const std::string& path);
void set_path(Node& root, const std::string& dotted, Node value);

std::string fmt_exact(double v);            // "%.17g", "null" when not finite
std::string fmt_fixed(double v, int decimals);  // "%.*f", no "-0", "null" when not finite
void json_escape(std::string& out, const std::string& s);
uint64_t fnv1a64(const std::string& s, uint64_t seed = 0xcbf29ce484222325ULL);
std::string hex16(uint64_t v);

}  // namespace dsd::cfg
