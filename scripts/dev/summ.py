import re, collections, sys
d = collections.OrderedDict()
for line in open(sys.argv[1]):
    m = re.match(r'(R=\d+ KB=\d+) (\S+) ([\d.]+)', line.replace('"',''))
    if m: d.setdefault(m.group(1), {})[m.group(2).split('.')[0]] = float(m.group(3))
for k, v in d.items():
    try:
        t = v['gpu__time_duration']/1e6; clk = v['sm__cycles_elapsed']/1e9
        print(f"{k:16s} t={t:6.2f}ms dram={v['dram__bytes_read']/1e9:6.1f}GB hit={v['lts__t_sector_hit_rate']:5.1f}% clk={clk:.2f}GHz tensor={v['sm__pipe_tensor_cycles_active']:5.1f}% cycles={t*clk:6.2f}M")
    except KeyError as e:
        print(k, 'missing', e)
